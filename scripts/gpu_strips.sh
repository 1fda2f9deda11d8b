# strip decomposition on virtual ranks (one GPU): tests with iteration counts
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r02_strips}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_strips.py tests/test_gpu_kernel_shapes.py -q -s -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc $?" >> $O/rc.txt
cat $O/rc.txt
