cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_float_nets_debug.py -m gpu -q -s > gpurun_out/dbg.log 2>&1
echo "rc=$?" >> gpurun_out/dbg.log
