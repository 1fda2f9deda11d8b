cd $GRAFT_REPO_ROOT
for T in 65536 16384 4096 1024 0; do
  echo "LDG_ROWS_BELOW=$T"
  LDG_ROWS_BELOW=$T timeout 300 python scripts/mg_times.py 256 ${MGP:-2,3,4}
done
