cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > $O/r3p_bench.json 2>$O/r3p_bench.err
timeout 900 python -m pytest tests/test_gpu_alexnet.py -m gpu -q -x -p no:hypothesispytest -k "bit_exact or fallback" > $O/r3p_tests.log 2>&1
echo "tests rc=$?" >> $O/r3p_tests.log
