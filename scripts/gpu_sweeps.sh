# level-0 sweep counts per degree: 20-step C2 bench of one degree per setting
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r02_sweeps}
mkdir -p $O
for P in ${PS:-4 3}; do
  for s in ${SETTINGS:-"0,0" "7,7" "6,8" "7,8" "5,7" "6,6"}; do
    pre=${s%,*}; post=${s#*,}
    if [ $pre = 0 ]; then unset LDG_MG_PRE0 LDG_MG_POST0; else export LDG_MG_PRE0=$pre LDG_MG_POST0=$post; fi
    timeout 300 python bench.py --no-cpu-baseline --no-clocks --p $P --steps 20 --warmup 5 > $O/b_${P}_${pre}_${post}.jsonl 2>/dev/null
    python - $O/b_${P}_${pre}_${post}.jsonl $P $s <<'PY'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); v=d['config']['per_p'][sys.argv[2]]
        print("p", sys.argv[2], "V(%s)"%sys.argv[3], "ms/step %.3f"%v['ms_per_step'], "its %.2f"%v['iterations_per_step'], "krylov %.3f"%v['ms_krylov'])
PY
  done
done
