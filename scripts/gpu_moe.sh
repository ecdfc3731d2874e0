cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_moe.py tests/test_gpu_alexnet.py -m gpu -q -x > gpurun_out/moe2_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/moe2_tests.log
python scripts/moe_profile.py > gpurun_out/moe2_prof.json 2> gpurun_out/moe2_prof.err
timeout 900 python bench.py --model alexnet_moe --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/moe2_bench.json 2> gpurun_out/moe2_bench.err
