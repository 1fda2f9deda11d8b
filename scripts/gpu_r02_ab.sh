# A/B: two-thread stage 1, p-coarsening chains; correctness subset first
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r02_ab}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernel_shapes.py tests/test_gpu_parity_scale.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc $?" >> $O/rc.txt
run() { name=$1; shift; env "$@" timeout 600 python bench.py --no-cpu-baseline --steps 5 > $O/$name.jsonl 2> $O/$name.err; echo "$name rc $?" >> $O/rc.txt; }
run base
run nohalf LDG_S1_HALF=5
run pc3_21 LDG_MG_PC3=2,1
run pc2_10 LDG_MG_PC2=1,0
run pc3_10 LDG_MG_PC3=1,0
run pc1_0 LDG_MG_PC1=0
cat $O/rc.txt
