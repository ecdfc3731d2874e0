# Quick check of the current code: AlexNet / MoE / executor parity tests + the default bench line.
cd $GRAFT_REPO_ROOT
TAG=${1:-q}
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_batch256.py tests/test_gpu_alexnet.py tests/test_gpu_executor_cpp.py tests/test_gpu_moe.py -m gpu -q -x -p no:hypothesispytest > $O/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> $O/${TAG}_tests.log
timeout 600 python bench.py --no-cpu-baseline > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
