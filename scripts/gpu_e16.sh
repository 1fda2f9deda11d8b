cd $GRAFT_REPO_ROOT
for E in 32 16; do
  echo "LDG_SMOOTHER_E=$E"
  LDG_SMOOTHER_E=$E timeout 300 python scripts/mg_times.py 256 2,3,4
  LDG_SMOOTHER_E=$E timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_e$E.log 2>&1
  python - $E <<'PY'
import json, sys
for line in open(f'gpurun_out/bench_e{sys.argv[1]}.log'):
    if line.startswith('{'):
        d = json.loads(line)
        print('value %.3e e2e %.3e' % (d['value'], d['e2e']['value']))
        for p, r in d['config']['per_p'].items():
            print(p, 'ms %.1f it %.1f' % (r['ms_per_step'], r['iterations_per_step']))
PY
done
timeout 900 python -m pytest tests/test_gpu_kernel_shapes.py tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -x 2>&1 | tail -3
