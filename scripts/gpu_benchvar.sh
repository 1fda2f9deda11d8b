cd $GRAFT_REPO_ROOT
show() { python -c "
import json,sys
for line in open('gpurun_out/bv.log'):
    if line.startswith('{'):
        d=json.loads(line); print(sys.argv[1], '  value %.3e' % d['value'], ' '.join('p%s %.1f' % (p, r['ms_per_step']) for p, r in d['config']['per_p'].items()))
" "$1"; }
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --p 0 > gpurun_out/bv.log 2>&1; show "p0 only"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --p 3 > gpurun_out/bv.log 2>&1; show "p3 only"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bv.log 2>&1; show "all"
LDG_TRACE_ITER=1 timeout 300 python scripts/step_breakdown.py 0,2,4 2>&1 | grep -v "^\[ldg trace\]" 
LDG_TRACE_ITER=1 timeout 300 python scripts/step_breakdown.py 0,2,4 2>&1 | grep "^\[ldg trace\]" | awk 'NR%9==5'
