cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_extrap5
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity_scale.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc $?" >> $O/rc.txt
run() { name=$1; shift; env "$@" timeout 600 python bench.py --no-cpu-baseline --steps 5 > $O/$name.jsonl 2> $O/$name.err; echo "$name rc $?" >> $O/rc.txt; }
run o4 LDG_EXTRAP=4
run o5 LDG_EXTRAP=5
cat $O/rc.txt
