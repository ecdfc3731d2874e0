cd $GRAFT_REPO_ROOT
O=gpurun_out
for D in 0 1 2; do QNB_FRONT_DBG=$D timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 > $O/r3r_dbg$D.json 2>/dev/null; done
timeout 900 python -m pytest tests/test_gpu_alexnet.py -m gpu -q -x -p no:hypothesispytest -k "bit_exact or fallback or dyn or resident" > $O/r3r_tests.log 2>&1
echo "tests rc=$?" >> $O/r3r_tests.log
