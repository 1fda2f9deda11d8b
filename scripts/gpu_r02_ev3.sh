# bjac staging change: tests subset, bench C2/C1/C5, p = 4 launch list
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r02_ev3}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernel_shapes.py tests/test_gpu_strips.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc $?" >> $O/rc.txt
timeout 900 python bench.py --no-cpu-baseline --steps 5 > $O/bench_c2.jsonl 2> $O/bench_c2.err; echo "c2 rc $?" >> $O/rc.txt
timeout 600 python bench.py --workload c1 --steps 20 > $O/bench_c1.jsonl 2> $O/bench_c1.err; echo "c1 rc $?" >> $O/rc.txt
timeout 1500 python bench.py --workload c5 --steps 3 --no-cpu-baseline > $O/bench_c5.jsonl 2> $O/bench_c5.err; echo "c5 rc $?" >> $O/rc.txt
timeout 600 python scripts/profile_step.py --p 4 --dim 256 --warmup 5 > $O/plain_p4.log 2>&1 && \
timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches_p4.csv python scripts/profile_step.py --p 4 --dim 256 --warmup 5 > $O/ncu_launch_p4.log 2>&1
echo "launch rc $?" >> $O/rc.txt
cat $O/rc.txt
