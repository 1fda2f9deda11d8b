cd $GRAFT_REPO_ROOT
O=gpurun_out/gs; mkdir -p $O
timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc $?" > $O/rc.txt
for r in 1 2; do for E in LDG_GS_HOST=1 LDG_GS_HOST=0; do
  env $E timeout 300 python scripts/step_breakdown.py 0,1,2,3,4 2>&1 | sed "s/^/[$E] /"
done; done > $O/ab.txt
cat $O/rc.txt; tail -3 $O/pytest.log; cat $O/ab.txt
