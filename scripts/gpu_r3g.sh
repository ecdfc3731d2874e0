cd $GRAFT_REPO_ROOT
O=gpurun_out
for D in 32 33 37; do QNB_FRONT_DBG=$D timeout 300 python bench.py --no-cpu-baseline --steps 3 --warmup 3 --profile-reps 1 > $O/r3g_dbg$D.json 2> $O/r3g_dbg$D.err; done
