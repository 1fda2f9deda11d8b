cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r02_ex5}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity_scale.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc $?" >> $O/rc.txt
run() { name=$1; shift; env "$@" timeout 900 python bench.py --no-cpu-baseline --no-clocks "$@" > $O/$name.jsonl 2> $O/$name.err; echo "$name rc $?" >> $O/rc.txt; }
runa() { name=$1; e=$2; shift 2; env $e timeout 900 python bench.py --no-cpu-baseline --no-clocks "$@" > $O/$name.jsonl 2> $O/$name.err; echo "$name rc $?" >> $O/rc.txt; }
runa pd5 LDG_EXTRAP=-1 --steps 5
runa o4s5 LDG_EXTRAP=4 --steps 5
runa pd20 LDG_EXTRAP=-1 --steps 20 --warmup 5
runa o4s20 LDG_EXTRAP=4 --steps 20 --warmup 5
cat $O/rc.txt
