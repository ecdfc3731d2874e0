cd $GRAFT_REPO_ROOT
TAG=${1:-r2i}
O=gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x -p no:hypothesispytest > $O/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> $O/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1
timeout 600 python bench.py > $O/${TAG}_int8.json 2> $O/${TAG}_int8.err
timeout 900 python bench.py --model alexnet_moe --steps 30 --warmup 5 > $O/${TAG}_moe.json 2> $O/${TAG}_moe.err
