cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_alexnet.py tests/test_gpu_batch256.py -m gpu -q -x -p no:hypothesispytest > $O/r3e_tests.log 2>&1
echo "tests rc=$?" >> $O/r3e_tests.log
for D in 0 1 2 3; do QNB_FRONT_DBG=$D timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > $O/r3e_dbg$D.json 2>/dev/null; done
QNB_FRONT_NO_SA=1 timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > $O/r3e_nosa.json 2>/dev/null
bash scripts/gpu_ncu_kernel.sh r3e_front front_kernel
