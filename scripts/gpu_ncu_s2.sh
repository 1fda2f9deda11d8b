# ncu --set full (with source) of the level-0 smoother kernels of one steady-state p = 4 step
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-ncu_s2}
mkdir -p $O
export LDG_S2_TMA=${LDG_S2_TMA:-0}
timeout 600 python scripts/profile_step.py --p 4 --dim 256 --warmup 5 > $O/plain_p4.log 2>&1 || { echo "plain p4 failed" >> $O/rc.txt; exit 1; }
timeout 1800 ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_s2f<\(int\)4, \(int\)1|k_s1f<\(int\)4|k_s2t<\(int\)4, \(int\)1" -c 4 -f -o $O/s2_p4 \
  python scripts/profile_step.py --p 4 --dim 256 --warmup 5 > $O/ncu_s2_p4.log 2>&1
echo "ncu rc $?" >> $O/rc.txt
cat $O/rc.txt
