cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_alexnet.py -m gpu -q -x -p no:hypothesispytest -k "bit_exact or fallback" > $O/r3f_tests.log 2>&1
echo "tests rc=$?" >> $O/r3f_tests.log
for D in 0 1 2 3 5 4 12 9; do QNB_FRONT_DBG=$D timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > $O/r3f_dbg$D.json 2>/dev/null; done
