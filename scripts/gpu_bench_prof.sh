cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py ${BENCH_ARGS:---steps 3 --warmup 3} > gpurun_out/bench.log 2>&1; echo "bench rc $?" >> gpurun_out/bench.log
python - <<'PY'
import json
for line in open('gpurun_out/bench.log'):
    if line.startswith('{'):
        d = json.loads(line)
        print('value %.3e e2e %.3e' % (d['value'], d['e2e']['value']))
        for p, r in d['config']['per_p'].items():
            print(p, 'ms %.1f it %.1f dofs %.3e' % (r['ms_per_step'], r['iterations_per_step'], r['dof_updates_per_s']))
        print('roof', d['roofline']['kernel'], '%.0f GB/s frac %.2f' % (d['roofline']['achieved'], d['roofline']['frac']))
        for p, o in d['roofline']['others'].items():
            print(p, 'asm %.0f spmv %.0f schur %.0f' % (o['assemble_GBps'], o['full_apply_compulsory_GBps'], o['schur_apply_GBps']))
PY
tail -1 gpurun_out/bench.log
for P in ${PS:-4}; do
timeout 600 python scripts/profile_step.py --p $P --dim 256 > gpurun_out/plain_p$P.log 2>&1 && \
timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_p$P.csv python scripts/profile_step.py --p $P --dim 256 > gpurun_out/ncu_p$P.log 2>&1
python scripts/ncu_summary.py gpurun_out/launches_p$P.csv > gpurun_out/launches_p${P}_summary.txt 2>&1
head -14 gpurun_out/launches_p${P}_summary.txt
tail -1 gpurun_out/plain_p$P.log
done
