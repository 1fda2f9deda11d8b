# Parity tests (all GPU tests), C3 launch list + bench line, C2 bench line.
cd $GRAFT_REPO_ROOT
O=gpurun_out/chk
mkdir -p $O
timeout 1200 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc $?" >> $O/pytest.log
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/c3_launches.csv python scripts/profile_step.py --blocks --p 4 --dim 1024 > $O/c3_ncu.log 2>&1
timeout 600 python bench.py --workload c3 --steps 10 > $O/bench_c3.jsonl 2> $O/bench_c3.err
timeout 900 python bench.py ${BENCH_ARGS:---steps 5 --warmup 3} > $O/bench_c2.jsonl 2> $O/bench_c2.err
tail -3 $O/pytest.log
for f in $O/bench_c3.jsonl $O/bench_c2.jsonl; do python -c "
import json,sys
d=json.loads([l for l in open('$f') if l.startswith('{')][-1]); print('$f', d['value'], d['ms_per_step'], d['roofline']['frac'])"; done
