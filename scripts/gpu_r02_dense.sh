# dense coarsest level: solver tests + bench with / without
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_dense
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernel_shapes.py tests/test_gpu_parity_scale.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc $?" >> $O/rc.txt
run() { name=$1; shift; env "$@" timeout 600 python bench.py --no-cpu-baseline --steps 5 > $O/$name.jsonl 2> $O/$name.err; echo "$name rc $?" >> $O/rc.txt; }
run dense
run off LDG_DENSE_MAX=0
run d400 LDG_DENSE_MAX=400
cat $O/rc.txt
