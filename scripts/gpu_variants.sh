# the same measurements against alternative builds (build/var_*/libldg_b200.so)
cd $GRAFT_REPO_ROOT
for V in base ${VARIANTS:-var_o4 var_o6 var_o8}; do
  if [ "$V" = base ]; then unset LDG_B200_LIB; else export LDG_B200_LIB=$PWD/build/$V/libldg_b200.so; fi
  echo "== $V"
  timeout 300 python scripts/mg_times.py 256 ${MGP:-2,4}
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline ${BARGS:---p 2,3,4} > gpurun_out/bench_$V.log 2>&1
  python - $V <<'PY'
import json, sys
for line in open(f'gpurun_out/bench_{sys.argv[1]}.log'):
    if line.startswith('{'):
        d = json.loads(line)
        print('  value %.3e' % d['value'], ' '.join('p%s %.1fms/%.1fit' % (p, r['ms_per_step'], r['iterations_per_step']) for p, r in d['config']['per_p'].items()))
PY
done
