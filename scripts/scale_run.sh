#!/bin/bash
# Strip-decomposition scaling runs on one node: one process
# per GPU over NCCL, launched the way the driver launches bench.py.
#   bash scripts/scale_run.sh [workload] [steps]      (default c5 3)
# weak: dim = 4096 sqrt(P/8) for C5 (1472, 2048, 2944, 4096), strong: 4096^2 fixed.
W=${1:-c5}
S=${2:-3}
mkdir -p gpurun_out/scale
NG=$(nvidia-smi -L | wc -l)
for N in 1 2 4 8; do
  [ "$N" -gt "$NG" ] && break
  for SC in strong weak; do
    if [ "$N" -eq 1 ]; then
      python bench.py --workload $W --steps $S --warmup 3 --scaling $SC --no-cpu-baseline \
        > gpurun_out/scale/${W}_${SC}_n$N.jsonl 2> gpurun_out/scale/${W}_${SC}_n$N.err
    else
      python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + N)) \
        bench.py --gpus $N --workload $W --steps $S --warmup 3 --scaling $SC \
        > gpurun_out/scale/${W}_${SC}_n$N.jsonl 2> gpurun_out/scale/${W}_${SC}_n$N.err
    fi
    echo "$W $SC N=$N rc $?"
  done
done
