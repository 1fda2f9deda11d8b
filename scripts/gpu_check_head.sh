# Validate HEAD on one B200: GPU tests, default bench, reference arm.
cd $GRAFT_REPO_ROOT
O=gpurun_out/head; mkdir -p $O
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/rc.txt
timeout 900 python bench.py > $O/bench_c2.jsonl 2> $O/bench_c2.err; echo "c2 rc $?" >> $O/rc.txt
tail -3 $O/pytest_gpu.log; cat $O/rc.txt
