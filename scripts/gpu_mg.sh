cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
[ -n "$SKIP_MG" ] || timeout 600 python scripts/mg_times.py 256 > gpurun_out/mg_times.log 2>&1; echo "rc $?" >> gpurun_out/mg_times.log
cat gpurun_out/mg_times.log
P=4 KREGEX="${KREGEX:-regex:k_stage2<|k_stage1<|k_stage1_rows<|k_stage2_rows<|k_bjac_axpy<|k_bjac_rows<}"
timeout 1800 ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "$KREGEX" -c ${NCOUNT:-22} -f -o gpurun_out/full2_p$P \
  python scripts/profile_step.py --p $P --dim 256 > gpurun_out/ncufull2_p$P.log 2>&1
echo "ncu rc $?"; tail -2 gpurun_out/ncufull2_p$P.log
