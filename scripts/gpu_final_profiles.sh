# Round-end evidence: bench lines (c2 default with the CPU baseline, c1, c3, c4, c5),
# the reference arm, ncu launch lists of one p=4 / p=2 step and one ncu --set full
# capture of the dominant kernels.  Everything lands in gpurun_out/final/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
O=gpurun_out/final
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_c2.jsonl 2> $O/bench_c2.err; echo "c2 rc $?" >> $O/rc.txt
timeout 600 python bench.py --impl reference > $O/bench_ref_c2.jsonl 2> $O/bench_ref_c2.err; echo "ref rc $?" >> $O/rc.txt
timeout 600 python bench.py --workload c1 --steps 20 > $O/bench_c1.jsonl 2> $O/bench_c1.err; echo "c1 rc $?" >> $O/rc.txt
timeout 900 python bench.py --workload c3 --steps 10 > $O/bench_c3.jsonl 2> $O/bench_c3.err; echo "c3 rc $?" >> $O/rc.txt
timeout 1500 python bench.py --workload c4 --steps 3 --no-cpu-baseline > $O/bench_c4.jsonl 2> $O/bench_c4.err; echo "c4 rc $?" >> $O/rc.txt
timeout 1500 python bench.py --workload c5 --steps 3 --no-cpu-baseline > $O/bench_c5.jsonl 2> $O/bench_c5.err; echo "c5 rc $?" >> $O/rc.txt
for P in 4 2; do
  timeout 600 python scripts/profile_step.py --p $P --dim 256 > $O/plain_p$P.log 2>&1 && \
  timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches_p$P.csv python scripts/profile_step.py --p $P --dim 256 > $O/ncu_launch_p$P.log 2>&1
  echo "launch p$P rc $?" >> $O/rc.txt
done
timeout 1800 ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_s2f<|k_s1f<|k_stage2<|k_stage1<|k_bjf<" -c 14 -f -o $O/full_p4 \
  python scripts/profile_step.py --p 4 --dim 256 > $O/ncu_full_p4.log 2>&1
echo "full rc $?" >> $O/rc.txt
cat $O/rc.txt
