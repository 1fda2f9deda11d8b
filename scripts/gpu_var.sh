cd $GRAFT_REPO_ROOT
show() { python -c "
import json,sys
for line in open('gpurun_out/bv.log'):
    if line.startswith('{'):
        d=json.loads(line); print(sys.argv[1], '  value %.3e' % d['value'], ' '.join('p%s %.1f' % (p, r['ms_per_step']) for p, r in d['config']['per_p'].items()))
" "$1"; }
for i in 1 2 3; do
  timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bv.log 2>&1; show "clocks  "
  timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-clocks > gpurun_out/bv.log 2>&1; show "noclocks"
done
