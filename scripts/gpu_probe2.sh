cd $GRAFT_REPO_ROOT
T=$1
for env in "X=1" "QNB_NO_PATCH=1" "QNB_NO_BSTAT=1" "QNB_NO_PATCH=1 QNB_NO_TMA=1"; do
  for d in 0 3; do env $env QNB_IGEMM_DBG=$d timeout 300 python scripts/igemm_probe.py | sed "s/^/$env /" >> gpurun_out/probe_$T.txt 2>> gpurun_out/probe_$T.err; done
done
