cd $GRAFT_REPO_ROOT
TAG=${1:-pt}
QNB_PATCH=1 timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_alexnet.py -m gpu -q -x -k "conv or alexnet" > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
for env in "QNB_PATCH=1" "X=1"; do
  for d in 0 3; do env $env QNB_IGEMM_DBG=$d timeout 300 python scripts/igemm_probe.py | sed "s/^/$env /" >> gpurun_out/${TAG}_probe.txt 2>> gpurun_out/${TAG}_probe.err; done
done
