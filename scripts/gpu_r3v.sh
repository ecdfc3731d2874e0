cd $GRAFT_REPO_ROOT
O=gpurun_out
for D in 0 1 3; do QNB_LIB_VARIANT=spin QNB_FRONT_DBG=$D timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 > $O/r3v_dbg$D.json 2>/dev/null; done
