cd $GRAFT_REPO_ROOT
O=gpurun_out
for D in 32 0; do QNB_LIB_VARIANT=spin QNB_FRONT_DBG=$D timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3 --profile-reps 1 > $O/r3j_spin$D.json 2> $O/r3j_spin$D.err; done
