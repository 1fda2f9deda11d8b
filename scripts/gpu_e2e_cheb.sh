cd $GRAFT_REPO_ROOT
O=gpurun_out/e2e; mkdir -p $O
timeout 300 python scripts/e2e_diag.py > $O/e2e.txt 2>&1
for C in 1 0; do for r in 1 2; do
  LDG_MG_CHEB=$C timeout 300 python scripts/step_breakdown.py 0,1,2,3,4 > $O/cheb$C.$r.txt 2>&1
done; done
cat $O/e2e.txt; head -50 $O/cheb*.txt
