# ncu --set full of the hot kernels of one steady-state p = 4 step (256^2) and
# of the degree-1 dense coarsest level at p = 2; the plain run must exit 0 first.
# The reports are summarised on the box (raw csv, details, table, traffic json)
# and removed: gpurun brings back at most 64 MiB.
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-ncu_full}
mkdir -p $O
timeout 600 python scripts/profile_step.py --p 4 --dim 256 --warmup 5 > $O/plain_p4.log 2>&1 || { echo "plain p4 failed" >> $O/rc.txt; exit 1; }
timeout 1800 ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_s2f<\(int\)4, \(int\)1|k_s1f<\(int\)4|k_stage2<\(int\)4|k_stage1<\(int\)4|k_stage1r<\(int\)4|k_dtrace<\(int\)4|k_bjac_warp<\(int\)4|k_assemble_rows<\(int\)4|k_full<\(int\)4" -c 20 -f -o $O/full_p4 \
  python scripts/profile_step.py --p 4 --dim 256 --warmup 5 > $O/ncu_full_p4.log 2>&1
echo "full p4 rc $?" >> $O/rc.txt
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_dense_gemv|k_s2f<\(int\)2, \(int\)1|k_s1f<\(int\)2|k_bjac_warp<\(int\)2|k_dense_col|k_s2_batch|k_s1_batch" -c 10 -f -o $O/full_p2 \
  python scripts/profile_step.py --p 2 --dim 256 --warmup 5 > $O/ncu_full_p2.log 2>&1
echo "full p2 rc $?" >> $O/rc.txt
for p in 4 2; do
  R=$O/full_p$p.ncu-rep
  [ -f $R ] || continue
  python scripts/ncu_table.py $R > $O/full_p${p}_table.txt
  ncu -i $R --page details --print-summary per-kernel > $O/full_p${p}_details.txt 2>/dev/null
  ncu -i $R --page raw --csv > $O/full_p${p}_raw.csv 2>/dev/null
  [ $p = 4 ] && python scripts/ncu_traffic.py $R $O/ncu_traffic.json 4 256 > $O/full_p4_traffic.txt
  rm -f $R
done
cat $O/rc.txt
