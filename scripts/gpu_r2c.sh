# GPU tests + AlexNet INT8 / FP16 / INT16 bench lines.
cd $GRAFT_REPO_ROOT
TAG=${1:-r2c}
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:hypothesispytest ${PYTEST_K:+-k "$PYTEST_K"} > $O/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> $O/${TAG}_tests.log
timeout 600 python bench.py > $O/${TAG}_int8.json 2> $O/${TAG}_int8.err
timeout 600 python bench.py --precision fp16 > $O/${TAG}_fp16.json 2> $O/${TAG}_fp16.err
timeout 600 python bench.py --precision int16 > $O/${TAG}_int16.json 2> $O/${TAG}_int16.err
