# Round-2 state check at HEAD: GPU tests, default bench, reference arm.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_head
mkdir -p $O
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider -x > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/rc.txt
timeout 900 python bench.py > $O/bench_c2.jsonl 2> $O/bench_c2.err; echo "c2 rc $?" >> $O/rc.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.jsonl 2> $O/bench_ref.err; echo "ref rc $?" >> $O/rc.txt
cat $O/rc.txt
