# multigrid parameter A/B at p = 3, 4 (5-step C2 bench, one degree per run)
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r02_tune}
mkdir -p $O
run() { name=$1; shift; env "$@" timeout 600 python bench.py --no-cpu-baseline --no-clocks --steps 5 --p 3,4 > $O/$name.jsonl 2> $O/$name.err; echo "$name rc $?" >> $O/rc.txt; }
run base
run l2_11 LDG_MG_PRE2=1 LDG_MG_POST2=1
run l2_21 LDG_MG_PRE2=2 LDG_MG_POST2=1
run l1_21 LDG_MG_PRE1=2 LDG_MG_POST1=1
run l1_22 LDG_MG_PRE1=2 LDG_MG_POST1=2
run r15 LDG_CHEB_RATIO=15
run r30 LDG_CHEB_RATIO=30
run s104 LDG_CHEB_SAFETY=1.04
run s112 LDG_CHEB_SAFETY=1.12
run v57 LDG_MG_PRE0=5 LDG_MG_POST0=7
run v77 LDG_MG_PRE0=7 LDG_MG_POST0=7
cat $O/rc.txt
