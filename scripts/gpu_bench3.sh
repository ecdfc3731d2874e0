cd $GRAFT_REPO_ROOT
TAG=${1:-b3}
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_alexnet.json 2> gpurun_out/${TAG}_alexnet.err
timeout 900 python bench.py --model alexnet_moe --steps 5 --warmup 3 > gpurun_out/${TAG}_moe.json 2> gpurun_out/${TAG}_moe.err
if [ -f tests/golden/vgg16_int8_calib.json ]; then
timeout 600 python bench.py --model vgg16 --batch 128 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_vgg.json 2> gpurun_out/${TAG}_vgg.err
fi
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err
