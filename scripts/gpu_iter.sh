# quick iteration: gpu tests (optionally a subset), multigrid timing, short bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest ${TESTS:-tests} -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
timeout 600 python scripts/mg_times.py 256 ${MGP:-0,1,2,3,4} > gpurun_out/mg_times.log 2>&1; echo "rc $?" >> gpurun_out/mg_times.log
cat gpurun_out/mg_times.log
timeout 900 python bench.py ${BENCH_ARGS:---steps 3 --warmup 3 --no-cpu-baseline} > gpurun_out/bench.log 2>&1; echo "bench rc $?" >> gpurun_out/bench.log
python - <<'PY'
import json
for line in open('gpurun_out/bench.log'):
    if line.startswith('{'):
        d = json.loads(line)
        print('value %.3e e2e %.3e' % (d['value'], d['e2e']['value']))
        for p, r in d['config']['per_p'].items():
            print(p, 'ms %.1f it %.1f dofs %.3e' % (r['ms_per_step'], r['iterations_per_step'], r['dof_updates_per_s']))
PY
tail -2 gpurun_out/bench.log
