cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "parity or fields" > gpurun_out/pytest_sel.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_sel.log
FULL=1 bash scripts/gpu_c3_prof.sh
KREGEX="k_s2f<|k_s1f<|k_stage2<|k_stage1<|k_bjf<" NCOUNT=14 TAG=full_s2f bash scripts/gpu_ncu_kernels.sh
tail -3 gpurun_out/pytest_sel.log
