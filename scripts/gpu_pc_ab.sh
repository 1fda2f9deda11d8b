# A/B of the p-coarsened multigrid level (LDG_MG_PC) on the C2 steps
cd $GRAFT_REPO_ROOT
O=gpurun_out/pc; mkdir -p $O
LDG_MG_PC=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "multigrid or c1_hundred or euler" > $O/pytest_pc1.log 2>&1; echo "pytest pc1 rc $?" >> $O/rc.txt
for r in 1 2; do
for E in "LDG_MG_PC=-1" "LDG_MG_PC=1" "LDG_MG_PC=0" "LDG_MG_PC=2"; do
  env $E timeout 300 python scripts/step_breakdown.py ${PS:-2,3,4} > "$O/$E.$r.txt" 2>&1
done; done
cat $O/rc.txt; tail -3 $O/pytest_pc1.log; for f in $O/LDG*.txt; do echo "== $f"; cat "$f"; done
