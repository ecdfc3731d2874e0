cd $GRAFT_REPO_ROOT
TAG=${1:-new}
timeout 300 python -m pytest tests/test_gpu_ops.py -k "conv or inner_product" -m gpu -q -x > gpurun_out/${TAG}_ops.log 2>&1
echo "ops rc=$?" >> gpurun_out/${TAG}_ops.log
timeout 900 python -m pytest tests/test_gpu_alexnet.py -m gpu -q -x > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
for d in 0 3; do QNB_IGEMM_DBG=$d timeout 300 python scripts/igemm_probe.py >> gpurun_out/${TAG}_probe.jsonl 2>> gpurun_out/${TAG}_probe.err; done
