cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r02_ex7}
mkdir -p $O
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/rc.txt
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench20.jsonl 2> $O/bench20.err; echo "bench20 rc $?" >> $O/rc.txt
timeout 1200 python scripts/tol_study.py 256 10 > $O/tol10.txt 2>&1; echo "tol rc $?" >> $O/rc.txt
cat $O/rc.txt
