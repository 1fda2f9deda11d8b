# A/B of alternative builds (build/variants/lib_*.so via LDG_B200_LIB) on step time
cd $GRAFT_REPO_ROOT
O=gpurun_out/var; mkdir -p $O
for r in 1 2; do for V in base ${VARIANTS:-s5 s6 s8 st6}; do
  if [ $V = base ]; then L=""; else L="LDG_B200_LIB=$GRAFT_REPO_ROOT/build/variants/lib_$V.so"; fi
  env $L timeout 300 python scripts/step_breakdown.py ${PS:-2,3,4} 2>&1 | sed "s/^/[$V] /"
done; done > $O/ab.txt
cat $O/ab.txt
