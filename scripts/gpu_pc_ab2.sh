# A/B of p-coarsening chains (LDG_MG_PC) per degree; 2 rounds each
cd $GRAFT_REPO_ROOT
O=gpurun_out/pc2; mkdir -p $O
run() {  # $1 = p list, rest = env
  local ps=$1; shift
  for r in 1 2; do env "$@" timeout 300 python scripts/step_breakdown.py $ps 2>&1 | sed "s/^/[$*] /"; done
}
{
run 4 LDG_MG_PC=-1
run 4 LDG_MG_PC=2
run 4 LDG_MG_PC=2,1
run 4 LDG_MG_PC=3,1
run 4 LDG_MG_PC=3,2,1
run 4 LDG_MG_PC=2,1 LDG_MG_PRE1=3 LDG_MG_POST1=2
run 4 LDG_MG_PC=2,1 LDG_MG_PRE1=2 LDG_MG_POST1=2
run 3 LDG_MG_PC=-1
run 3 LDG_MG_PC=1
run 3 LDG_MG_PC=2,1
run 3 LDG_MG_PC=2
run 3 LDG_MG_PC=1 LDG_MG_PRE1=3 LDG_MG_POST1=2
run 2 LDG_MG_PC=-1
run 2 LDG_MG_PC=1
run 2 LDG_MG_PC=1 LDG_MG_PRE1=3 LDG_MG_POST1=2
run 2 LDG_MG_PC=0
} > $O/ab.txt
cat $O/ab.txt
