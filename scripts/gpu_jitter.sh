cd $GRAFT_REPO_ROOT
O=gpurun_out/jit; mkdir -p $O
{ nproc; lscpu | grep -i "numa\|model name\|socket"; nvidia-smi topo -m; } > $O/host.txt 2>&1
for r in 1 2 3 4 5 6; do
  LDG_TRACE_ITER=1 timeout 120 python scripts/step_breakdown.py 0,4 > $O/t$r.txt 2>&1
  echo "run $r cpu $(taskset -pc $$ 2>/dev/null)" >> $O/t$r.txt
done
for r in 1 2 3; do
  LDG_TRACE_ITER=1 timeout 120 taskset -c 0-7 python scripts/step_breakdown.py 0,4 > $O/pin$r.txt 2>&1
done
cat $O/host.txt; for f in $O/t*.txt $O/pin*.txt; do echo "== $f"; grep -v "^\[ldg trace\]" $f; grep "^\[ldg trace\]" $f | tail -2; done
