# BASELINE config 3 (1024^2, p = 4, assembly only): plain timing, the ncu launch
# list of one assemble_blocks call and a --set full capture of its kernels.
cd $GRAFT_REPO_ROOT
O=gpurun_out/c3${TAG:+_$TAG}
mkdir -p $O
timeout 300 python scripts/profile_step.py --blocks --p 4 --dim 1024 --warmup 4 > $O/plain.log 2>&1; echo "plain rc $?" >> $O/rc.txt
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/launches.csv python scripts/profile_step.py --blocks --p 4 --dim 1024 > $O/ncu_launch.log 2>&1; echo "launch rc $?" >> $O/rc.txt
if [ -n "$FULL" ]; then
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled \
  -c 4 -f -o $O/full python scripts/profile_step.py --blocks --p 4 --dim 1024 > $O/ncu_full.log 2>&1; echo "full rc $?" >> $O/rc.txt
fi
cat $O/rc.txt; cat $O/plain.log | tail -3
