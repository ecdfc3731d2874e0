cd $GRAFT_REPO_ROOT
TAG=${1:-vgg}
timeout 900 python -m pytest tests/test_gpu_float_nets.py -k vgg16_int8_full -m gpu -q -x > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
timeout 600 python bench.py --model vgg16 --batch 128 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
