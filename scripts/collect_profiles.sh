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
[ -d $F/ncu ] && N=$F/ncu
# summaries written on the GPU box by scripts/gpu_ncu_full.sh
for p in 4 2; do
  [ -f $N/full_p${p}_table.txt ] && cp $N/full_p${p}_table.txt $P/${R}_ncu_full_p${p}_table.txt
  [ -f $N/full_p${p}_details.txt ] && cp $N/full_p${p}_details.txt $P/${R}_ncu_full_p${p}_details.txt
done
[ -f $N/full_p4_traffic.txt ] && cp $N/full_p4_traffic.txt $P/${R}_ncu_full_p4_traffic.txt
[ -f $N/ncu_traffic.json ] && cp $N/ncu_traffic.json $P/${R}_ncu_traffic.json
ls -la $P | tail -30
