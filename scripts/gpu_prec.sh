cd $GRAFT_REPO_ROOT
O=gpurun_out
TAG=${1:-prec}
timeout 300 python bench.py --no-cpu-baseline > $O/${TAG}_int8.json 2>/dev/null
timeout 300 python bench.py --precision fp16 --no-cpu-baseline > $O/${TAG}_fp16.json 2>/dev/null
timeout 300 python bench.py --precision int16 --no-cpu-baseline > $O/${TAG}_int16.json 2>/dev/null
