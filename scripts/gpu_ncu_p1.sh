# ncu --set full (with source) of the degree-1 smoother kernels of one steady-state p = 1 step
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-ncu_p1}
mkdir -p $O
timeout 600 python scripts/profile_step.py --p 1 --dim 256 --warmup 5 > $O/plain_p1.log 2>&1 || { echo "plain failed" >> $O/rc.txt; exit 1; }
timeout 1800 ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_s2f<\(int\)1, \(int\)1|k_s1f<\(int\)1" -c 6 -f -o $O/p1 \
  python scripts/profile_step.py --p 1 --dim 256 --warmup 5 > $O/ncu_p1.log 2>&1
echo "ncu rc $?" >> $O/rc.txt
cat $O/rc.txt
