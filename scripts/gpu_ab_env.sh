# A/B of an environment switch: ENVA / ENVB (e.g. "LDG_PDL=0" / "LDG_PDL=1")
cd $GRAFT_REPO_ROOT
for E in "$ENVA" "$ENVB"; do
  echo "== $E"
  env $E timeout 300 python scripts/mg_times.py 256 ${MGP:-0,2,4}
  env $E timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline ${BARGS:-} > gpurun_out/bench_ab.log 2>&1
  python - <<'PY'
import json
for line in open('gpurun_out/bench_ab.log'):
    if line.startswith('{'):
        d = json.loads(line)
        print('  value %.3e' % d['value'], ' '.join('p%s %.1fms/%.1fit' % (p, r['ms_per_step'], r['iterations_per_step']) for p, r in d['config']['per_p'].items()))
PY
done
