# ncu --set full of selected kernels of one profiled step (p=$P, dim 256)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P=${P:-4}
timeout 600 python scripts/profile_step.py --p $P --dim 256 > gpurun_out/plain_sel_p$P.log 2>&1 && \
timeout 1800 ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:${KREGEX}" -c ${NCOUNT:-6} -f -o gpurun_out/${TAG:-sel}_p$P \
  python scripts/profile_step.py --p $P --dim 256 > gpurun_out/ncu_sel_p$P.log 2>&1
echo "ncu rc $?"; tail -2 gpurun_out/ncu_sel_p$P.log
