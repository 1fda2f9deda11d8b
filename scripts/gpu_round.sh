# tests, bench, launch list, full capture
cd $GRAFT_REPO_ROOT
bash scripts/gpu_full.sh
bash scripts/gpu_ncu_full.sh
