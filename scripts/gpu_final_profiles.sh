# Round-end evidence: GPU tests, bench lines (C2 default with the CPU baseline,
# C1, C3, C4, C5), the reference arm, ncu launch lists of one steady-state p = 4
# / p = 2 step and ncu --set full captures of the hot kernels.  Everything lands
# in gpurun_out/${1:-final}/ (copy into profiles/ with scripts/collect_profiles.sh).
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-final}
mkdir -p $O
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/rc.txt
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_c2.jsonl 2> $O/bench_c2.err; echo "c2 rc $?" >> $O/rc.txt
timeout 600 python bench.py --workload c1 --steps 20 > $O/bench_c1.jsonl 2> $O/bench_c1.err; echo "c1 rc $?" >> $O/rc.txt
timeout 900 python bench.py --workload c3 --steps 10 > $O/bench_c3.jsonl 2> $O/bench_c3.err; echo "c3 rc $?" >> $O/rc.txt
timeout 1500 python bench.py --workload c4 --steps 3 --no-cpu-baseline > $O/bench_c4.jsonl 2> $O/bench_c4.err; echo "c4 rc $?" >> $O/rc.txt
timeout 1500 python bench.py --workload c5 --steps 3 --no-cpu-baseline > $O/bench_c5.jsonl 2> $O/bench_c5.err; echo "c5 rc $?" >> $O/rc.txt
for P in 4 3 2; do
  timeout 600 python scripts/profile_step.py --p $P --dim 256 --warmup 5 > $O/plain_p$P.log 2>&1 && \
  timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches_p$P.csv python scripts/profile_step.py --p $P --dim 256 --warmup 5 > $O/ncu_launch_p$P.log 2>&1
  echo "launch p$P rc $?" >> $O/rc.txt
done
bash scripts/gpu_ncu_full.sh ${1:-final}/ncu
timeout 1200 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_c2.jsonl 2> $O/bench_ref_c2.err; echo "ref rc $?" >> $O/rc.txt
cat $O/rc.txt
