cd $GRAFT_REPO_ROOT
TAG=${1:-r2g}
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:hypothesispytest -k "moe or device_resident or batch256 or inner_product" > $O/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> $O/${TAG}_tests.log
timeout 600 python bench.py --no-cpu-baseline > $O/${TAG}_int8.json 2> $O/${TAG}_int8.err
timeout 900 python bench.py --model alexnet_moe --steps 30 --warmup 5 > $O/${TAG}_moe.json 2> $O/${TAG}_moe.err
