# full GPU test suite + the driver's bench command
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r02_check}
mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/rc.txt
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_c2.jsonl 2> $O/bench_c2.err; echo "c2 rc $?" >> $O/rc.txt
tail -3 $O/pytest_gpu.log
cat $O/rc.txt
