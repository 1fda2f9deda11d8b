# quick check of an operator / smoother change: timing, the parity + shape + strip tests, a 10-step bench
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r02_quick}
mkdir -p $O
timeout 300 python scripts/mg_times.py 256 ${PS:-0,1,2,3,4} > $O/mg.txt 2>&1; grep "^p=" $O/mg.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernel_shapes.py tests/test_gpu_parity_scale.py tests/test_gpu_strips.py tests/test_gpu_exports.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc $?" >> $O/rc.txt
tail -3 $O/pytest.log
timeout 600 python bench.py --no-cpu-baseline --steps 10 > $O/bench.jsonl 2> $O/bench.err; echo "bench rc $?" >> $O/rc.txt
python - $O/bench.jsonl <<'PY'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print("bench", round(d['ms_per_step'],2), {p:(round(v['ms_per_step'],2),v['iterations_per_step'],'%.1e'%v['max_residual']) for p,v in d['config']['per_p'].items()})
        print({p:round(v['schur_apply_GBps']) for p,v in d['roofline']['others'].items()})
PY
cat $O/rc.txt
