# A/B of the assembly kernels (row form vs LDG_ASM_V1=1) on BASELINE config 3,
# parity tests, and a C2 bench line.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/asm
O=gpurun_out/asm
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc $?" >> $O/pytest.log
for v in 0 1; do
  LDG_ASM_V1=$v timeout 300 python scripts/profile_step.py --blocks --p 4 --dim 1024 --warmup 4 > $O/c3_v$v.log 2>&1
  for p in 2 3; do LDG_ASM_V1=$v timeout 300 python scripts/profile_step.py --blocks --p $p --dim 1024 --warmup 3 > $O/c3_p${p}_v$v.log 2>&1; done
done
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/launches.csv python scripts/profile_step.py --blocks --p 4 --dim 1024 > $O/ncu_launch.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:k_assemble -c 1 -f -o $O/full python scripts/profile_step.py --blocks --p 4 --dim 1024 > $O/ncu_full.log 2>&1
timeout 600 python bench.py --workload c3 --steps 5 > $O/bench_c3.jsonl 2>&1
tail -2 $O/pytest.log; grep profiled $O/c3*.log
