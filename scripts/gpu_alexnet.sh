cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_alexnet.py -m gpu -q -x > gpurun_out/g2_alex.log 2>&1
echo "alex rc=$?" >> gpurun_out/g2_alex.log
