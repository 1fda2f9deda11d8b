# grid-cooperative multigrid tail: GPU tests of the solver paths, C2 bench, tolerance study
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_tail
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernel_shapes.py tests/test_gpu_parity_scale.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc $?" >> $O/rc.txt
timeout 600 python bench.py --no-cpu-baseline > $O/bench_c2.jsonl 2> $O/bench_c2.err; echo "c2 rc $?" >> $O/rc.txt
LDG_TAIL_MAXK=0 timeout 600 python bench.py --no-cpu-baseline --steps 3 > $O/bench_c2_notail.jsonl 2> $O/bench_c2_notail.err; echo "c2 notail rc $?" >> $O/rc.txt
timeout 900 python scripts/tol_study.py 256 3 > $O/tol.txt 2>&1; echo "tol rc $?" >> $O/rc.txt
cat $O/rc.txt
