cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_extrap2
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity_scale.py -q -x -p no:cacheprovider -k "extrapolated or c2_default" > $O/pytest.log 2>&1; echo "pytest rc $?" >> $O/rc.txt
timeout 600 python bench.py --no-cpu-baseline > $O/bench.jsonl 2> $O/bench.err; echo "bench rc $?" >> $O/rc.txt
cat $O/rc.txt
