cd $GRAFT_REPO_ROOT
TAG=${1:-new}
timeout 900 python -m pytest tests/test_gpu_ops.py -k "conv" -m gpu -q -x > gpurun_out/${TAG}_ops.log 2>&1
echo "ops rc=$?" >> gpurun_out/${TAG}_ops.log
timeout 900 python -m pytest tests/test_gpu_moe.py tests/test_gpu_executor_cpp.py -m gpu -q -x -s > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
