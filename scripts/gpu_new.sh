cd $GRAFT_REPO_ROOT
TAG=${1:-new}
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_alexnet.py tests/test_gpu_float_nets.py tests/test_gpu_moe.py -m gpu -q -x -k "not vgg16_int8_full" > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
