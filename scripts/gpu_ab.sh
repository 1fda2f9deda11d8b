# A/B of environment switches on the in-tree library: multigrid / operator timing
# (scripts/mg_times.py) and a 10-step C2 bench per setting, e.g.
#   gpurun -- 'bash scripts/gpu_ab.sh r02_ab "LDG_RANK_FORM=0"'
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r02_ab}
mkdir -p $O
shift
i=0
for setting in "" "$@"; do
  name=$([ -z "$setting" ] && echo base || echo v$i)
  echo "== $name $setting"
  env $setting timeout 300 python scripts/mg_times.py 256 ${PS:-0,1,2,3,4} > $O/mg_$name.txt 2>&1; echo "mg $name rc $?" >> $O/rc.txt
  grep -A1 "^p=" $O/mg_$name.txt
  env $setting timeout 600 python bench.py --no-cpu-baseline --steps 10 > $O/bench_$name.jsonl 2> $O/bench_$name.err; echo "bench $name rc $?" >> $O/rc.txt
  i=$((i+1))
done
cat $O/rc.txt
