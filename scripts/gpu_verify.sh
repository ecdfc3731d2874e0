# Round-end verification: GPU tests, smoke, default bench line, reference arm, MoE / VGG lines.
cd $GRAFT_REPO_ROOT
TAG=${1:-ver}
timeout 1200 python -m pytest tests -m gpu -q -x -p no:hypothesispytest > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err
timeout 900 python bench.py --model alexnet_moe --steps 30 --warmup 5 > gpurun_out/${TAG}_moe.json 2> gpurun_out/${TAG}_moe.err
timeout 900 python bench.py --model vgg16 --batch 128 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_vgg.json 2> gpurun_out/${TAG}_vgg.err
