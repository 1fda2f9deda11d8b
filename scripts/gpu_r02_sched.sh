# setup overlap on/off and level-0 sweep schedules with the extrapolated start
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_sched
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernel_shapes.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc $?" >> $O/rc.txt
run() { name=$1; shift; env "$@" timeout 600 python bench.py --no-cpu-baseline --steps 5 > $O/$name.jsonl 2> $O/$name.err; echo "$name rc $?" >> $O/rc.txt; }
run ov
run noov LDG_SETUP_OVERLAP=0
for s in "4 6" "5 6" "4 5" "6 7" "3 5"; do set -- $s; run pre$1post$2 LDG_MG_PRE0=$1 LDG_MG_POST0=$2; done
cat $O/rc.txt
