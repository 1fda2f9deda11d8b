cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r02_tune2}
mkdir -p $O
run() { name=$1; shift; env "$@" timeout 600 python bench.py --no-cpu-baseline --no-clocks --steps 5 > $O/$name.jsonl 2> $O/$name.err; echo "$name rc $?" >> $O/rc.txt; }
run base
run s104 LDG_CHEB_SAFETY=1.04
run s100 LDG_CHEB_SAFETY=1.00
run s104l2 LDG_CHEB_SAFETY=1.04 LDG_MG_PRE2=1 LDG_MG_POST2=1
run base2
cat $O/rc.txt
