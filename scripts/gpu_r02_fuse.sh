# coarse-level phase fusion variants: V-cycle / step times per degree
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_fuse
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernel_shapes.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc $?" >> $O/rc.txt
run() { name=$1; shift; env "$@" timeout 600 python bench.py --no-cpu-baseline --steps 3 > $O/$name.jsonl 2> $O/$name.err; echo "$name rc $?" >> $O/rc.txt; }
run A
run B LDG_TAIL_MAXK=0
run C LDG_TAIL_MAXK=0 LDG_FUSE_S1=2 LDG_FUSE_S1_MAXK=32768
run D LDG_FUSE_S1=2 LDG_FUSE_S1_MAXK=32768
run E LDG_TAIL_MAXK=0 LDG_FUSE_SMALL=0
cat $O/rc.txt
