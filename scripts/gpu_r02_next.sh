# new general-mesh multigrid test, GPU test suite subset, bench + p-coarsening A/B
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r02_next}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity_scale.py -q -s -x -p no:cacheprovider -k "general_mesh or extrapolated" > $O/pytest_new.log 2>&1; echo "pytest new rc $?" >> $O/rc.txt
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/rc.txt
timeout 600 python bench.py --no-cpu-baseline --steps 5 > $O/bench.jsonl 2> $O/bench.err; echo "bench rc $?" >> $O/rc.txt
LDG_MG_PC4=21 timeout 600 python bench.py --no-cpu-baseline --steps 5 --p 4 > $O/pc21.jsonl 2> $O/pc21.err; echo "pc21 rc $?" >> $O/rc.txt
cat $O/rc.txt
