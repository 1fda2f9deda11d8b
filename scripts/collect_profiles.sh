#!/bin/bash
# Copy the round-end evidence from gpurun_out/<dir> (scripts/gpu_final_profiles.sh <dir>)
# into profiles/ under the round prefix: bash scripts/collect_profiles.sh r02 gpurun_out/r02_ev1
R=${1:-r02}
F=${2:-gpurun_out/final}
P=profiles
set -e
for w in c2 ref_c2 c1 c3 c4 c5; do
  [ -f $F/bench_$w.jsonl ] && grep '^{' $F/bench_$w.jsonl > $P/${R}_bench_final_$w.jsonl || true
done
cp $F/pytest_gpu.log $P/${R}_pytest_gpu_final.log
cp $F/gpu.txt $P/${R}_gpu.txt
for p in 4 3 2; do
  if [ -f $F/launches_p$p.csv ]; then
    python scripts/ncu_summary.py $F/launches_p$p.csv > $P/${R}_launches_final_p${p}_summary.txt
    python scripts/ncu_by_grid.py $F/launches_p$p.csv > $P/${R}_launches_final_p${p}_by_grid.txt
    cp $F/launches_p$p.csv $P/${R}_launches_final_p$p.csv
    cp $F/plain_p$p.log $P/${R}_launches_final_p${p}_step.log
  fi
done
N=$F
[ -f $F/ncu/full_p4.ncu-rep ] && N=$F/ncu
if [ -f $N/full_p4.ncu-rep ]; then
  python scripts/ncu_traffic.py $N/full_p4.ncu-rep $P/${R}_ncu_traffic.json 4 256 > $P/${R}_ncu_full_p4_traffic.txt
  python scripts/ncu_table.py $N/full_p4.ncu-rep > $P/${R}_ncu_full_p4_table.txt
  ncu -i $N/full_p4.ncu-rep --page details --print-summary per-kernel > $P/${R}_ncu_full_p4_details.txt 2>/dev/null || true
fi
if [ -f $N/full_p2.ncu-rep ]; then
  python scripts/ncu_table.py $N/full_p2.ncu-rep > $P/${R}_ncu_full_p2_table.txt
  ncu -i $N/full_p2.ncu-rep --page details --print-summary per-kernel > $P/${R}_ncu_full_p2_details.txt 2>/dev/null || true
fi
ls -la $P | tail -30
