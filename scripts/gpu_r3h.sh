cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_alexnet.py -m gpu -q -x -p no:hypothesispytest -k "bit_exact or fallback" > $O/r3h_tests.log 2>&1
echo "tests rc=$?" >> $O/r3h_tests.log
for D in 0 1 2 3 5; do QNB_FRONT_DBG=$D timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > $O/r3h_dbg$D.json 2>/dev/null; done
for D in 32 34; do QNB_FRONT_DBG=$D timeout 300 python bench.py --no-cpu-baseline --steps 3 --warmup 3 --profile-reps 1 > $O/r3h_dbg$D.json 2> $O/r3h_dbg$D.err; done
