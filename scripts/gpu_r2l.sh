cd $GRAFT_REPO_ROOT
TAG=${1:-r2l}
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:hypothesispytest -k "alexnet or batch256 or executor or moe_int8 or convsweep" > $O/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> $O/${TAG}_tests.log
bash scripts/gpu_ab_env.sh $TAG "X=0" "QNB_NO_SLAB=1"
