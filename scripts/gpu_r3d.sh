cd $GRAFT_REPO_ROOT
bash scripts/gpu_ncu_kernel.sh r3d_front front_kernel
bash scripts/gpu_ncu_kernel.sh r3d_lrn pool_lrn5
# phase probes: epilogue math off (1), MMAs off (2)
for D in 1 2 3; do QNB_FRONT_DBG=$D timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/r3d_dbg$D.json 2>/dev/null; done
