cd $GRAFT_REPO_ROOT
TAG=${1:-r2j}
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:hypothesispytest -k "alexnet or batch256 or executor or moe_int8 or conv_int8" > $O/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> $O/${TAG}_tests.log
bash scripts/gpu_ab_env.sh $TAG "X=0" "QNB_NO_PPATCH=1" "QNB_HK_1COPY=1"
