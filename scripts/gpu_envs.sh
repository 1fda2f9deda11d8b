# mg_times + bench under several environment settings (ENVS, ';'-separated)
cd $GRAFT_REPO_ROOT
IFS=';' read -ra LIST <<< "$ENVS"
for E in "${LIST[@]}"; do
  echo "== $E"
  env $E timeout 300 python scripts/mg_times.py 256 ${MGP:-2,4} | grep -v "^$"
  env $E timeout 600 python bench.py --steps ${BSTEPS:-2} --warmup 2 --no-cpu-baseline ${BARGS:-} > gpurun_out/bench_envs.log 2>&1
  python - <<'PY'
import json
for line in open('gpurun_out/bench_envs.log'):
    if line.startswith('{'):
        d = json.loads(line)
        print('  value %.3e' % d['value'], ' '.join('p%s %.1fms/%.1fit' % (p, r['ms_per_step'], r['iterations_per_step']) for p, r in d['config']['per_p'].items()))
PY
done
