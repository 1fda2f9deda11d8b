# tensor-core stage 1 (k_s1t) against the FP32 FMA kernel (k_s1f)
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_s1tc
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernel_shapes.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc $?" >> $O/rc.txt
run() { name=$1; shift; env "$@" timeout 600 python bench.py --no-cpu-baseline --steps 3 > $O/$name.jsonl 2> $O/$name.err; echo "$name rc $?" >> $O/rc.txt; }
run tc
run off LDG_S1_TC=5
run tc1 LDG_S1_TC=1
cat $O/rc.txt
