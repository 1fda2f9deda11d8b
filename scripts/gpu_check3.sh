# All GPU tests, C2 and C4 bench lines.
cd $GRAFT_REPO_ROOT
O=gpurun_out/chk3
mkdir -p $O
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc $?" >> $O/pytest.log
timeout 900 python bench.py --no-cpu-baseline > $O/bench_c2.jsonl 2> $O/bench_c2.err
timeout 1500 python bench.py --workload c4 --steps 3 --no-cpu-baseline > $O/bench_c4.jsonl 2> $O/bench_c4.err
tail -3 $O/pytest.log
for f in c2 c4; do python -c "
import json
d=json.loads([l for l in open('$O/bench_$f.jsonl') if l.startswith('{')][-1])
pp=' '.join('p%s %.1f/%.1f'%(p,v['ms_per_step'],v['iterations_per_step']) for p,v in d['config']['per_p'].items())
print('$f', '%.4g'%d['value'], '%.2f'%d['ms_per_step'], 'e2e %.4g'%d['e2e']['value'], pp)"; done
