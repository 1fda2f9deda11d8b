# V-cycle parameter sweep (environment overrides), bench p=$PS
cd $GRAFT_REPO_ROOT
while read -r E; do
  [ -z "$E" ] && continue
  env $E timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --p ${PS:-2,4} > gpurun_out/bench_tune.log 2>&1
  python - "$E" <<'PY'
import json, sys
for line in open('gpurun_out/bench_tune.log'):
    if line.startswith('{'):
        d = json.loads(line)
        print('%-60s' % sys.argv[1], ' '.join('p%s %6.1fms/%5.1fit' % (p, r['ms_per_step'], r['iterations_per_step']) for p, r in d['config']['per_p'].items()), flush=True)
PY
done <<'LIST'
LDG_MG_THETA=1
LDG_MG_THETA=0.8
LDG_MG_THETA=1.2
LDG_MG_THETA=1.4
LDG_MG_THETA=1.7
LDG_MG_THETA=1.4 LDG_MG_SMOOTHER=rb LDG_MG_OMEGA_GS=0.9
LIST
