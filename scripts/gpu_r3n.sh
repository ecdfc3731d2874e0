cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_alexnet.py tests/test_gpu_batch256.py -m gpu -q -x -p no:hypothesispytest > $O/r3n_tests.log 2>&1
echo "tests rc=$?" >> $O/r3n_tests.log
timeout 300 python bench.py --no-cpu-baseline > $O/r3n_bench.json 2>$O/r3n_bench.err
QNB_NO_FRONT_PACK=1 timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > $O/r3n_nopack.json 2>/dev/null
