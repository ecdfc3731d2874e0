cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 > $O/r3q_bench.json 2>$O/r3q_bench.err
timeout 1500 python -m pytest tests/test_gpu_alexnet.py tests/test_gpu_batch256.py tests/test_gpu_ops.py tests/test_gpu_float_nets.py -m gpu -q -x -p no:hypothesispytest > $O/r3q_tests.log 2>&1
echo "tests rc=$?" >> $O/r3q_tests.log
