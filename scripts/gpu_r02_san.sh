cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_san
mkdir -p $O
timeout 300 python scripts/dense_dbg.py 64 0,1,2,3,4 > $O/plain.log 2>&1; echo "plain rc $?" >> $O/rc.txt
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/dense_dbg.py 64 0,4 > $O/memcheck.log 2>&1; echo "memcheck rc $?" >> $O/rc.txt
cat $O/rc.txt
