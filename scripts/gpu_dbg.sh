cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_ops.py -m gpu -q -k "tiling_and_split" > gpurun_out/dbg.log 2>&1
echo "rc=$?" >> gpurun_out/dbg.log
