# operator / smoother kernels A/B: multigrid + operator timing, correctness subset
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r02_rank}
mkdir -p $O
mg() { name=$1; shift; env "$@" timeout 300 python scripts/mg_times.py 256 ${PS:-0,1,2,3,4} > $O/mg_$name.txt 2>&1; echo "mg $name rc $?" >> $O/rc.txt; echo "== $name"; grep -A1 "^p=" $O/mg_$name.txt; }
mg new
mg tables LDG_RANK_FORM=0
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernel_shapes.py tests/test_gpu_parity_scale.py tests/test_gpu_strips.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc $?" >> $O/rc.txt
tail -5 $O/pytest.log
run() { name=$1; shift; env "$@" timeout 600 python bench.py --no-cpu-baseline --steps 10 > $O/$name.jsonl 2> $O/$name.err; echo "$name rc $?" >> $O/rc.txt; }
run bench_new
run bench_tables LDG_RANK_FORM=0
cat $O/rc.txt
