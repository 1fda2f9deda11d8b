# A/B of library build variants (build/var/lib*.so, LDG_B200_LIB): multigrid timing + 10-step bench
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r02_var}
mkdir -p $O
for v in base ${VARIANTS:-a b c d e}; do
  if [ $v = base ]; then unset LDG_B200_LIB; else export LDG_B200_LIB=$GRAFT_REPO_ROOT/build/var/lib$v.so; fi
  timeout 300 python scripts/mg_times.py 256 ${PS:-3,4} > $O/mg_$v.txt 2>&1; echo "mg $v rc $?" >> $O/rc.txt
  echo "== $v"; grep -A1 "^p=" $O/mg_$v.txt
  timeout 600 python bench.py --no-cpu-baseline --steps 10 > $O/bench_$v.jsonl 2> $O/bench_$v.err; echo "bench $v rc $?" >> $O/rc.txt
  python - $O/bench_$v.jsonl <<'PY'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print("   bench", round(d['ms_per_step'],2), {p:(round(v['ms_per_step'],2),v['iterations_per_step']) for p,v in d['config']['per_p'].items()})
PY
done
cat $O/rc.txt
