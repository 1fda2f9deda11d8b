# one `ncu --set full` capture of the top kernels of one profiled step (p=$P, dim 256)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P=${P:-4}
timeout 600 python scripts/profile_step.py --p $P --dim 256 > gpurun_out/plainfull_p$P.log 2>&1 && \
timeout 1800 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k "regex:${KREGEX:-k_stage|k_assemble|k_bjac|k_full}" -c ${NCOUNT:-8} -f -o gpurun_out/full_p$P \
  python scripts/profile_step.py --p $P --dim 256 > gpurun_out/ncufull_p$P.log 2>&1
echo "ncu full rc $?"
tail -3 gpurun_out/ncufull_p$P.log
