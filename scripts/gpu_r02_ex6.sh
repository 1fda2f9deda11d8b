cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r02_ex6}
mkdir -p $O
runa() { name=$1; e=$2; shift 2; env $e timeout 900 python bench.py --no-cpu-baseline --no-clocks "$@" > $O/$name.jsonl 2> $O/$name.err; echo "$name rc $?" >> $O/rc.txt; }
for o in 3 4 5 6 7 8; do runa o$o LDG_EXTRAP=$o --steps 20 --warmup 5; done
cat $O/rc.txt
