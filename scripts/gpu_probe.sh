cd $GRAFT_REPO_ROOT
for d in 0 1 2 3; do QNB_IGEMM_DBG=$d timeout 300 python scripts/igemm_probe.py >> gpurun_out/probe_$1.jsonl 2>> gpurun_out/probe_$1.err; done
