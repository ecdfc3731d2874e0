cd $GRAFT_REPO_ROOT
O=gpurun_out
for D in 99 97; do QNB_FRONT_DBG=$D timeout 300 python bench.py --no-cpu-baseline --steps 3 --warmup 3 --profile-reps 1 > $O/r3w_dbg$D.json 2> $O/r3w_dbg$D.err; done
for D in 67 65; do QNB_FRONT_DBG=$D timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > $O/r3w_b$D.json 2> /dev/null; done
