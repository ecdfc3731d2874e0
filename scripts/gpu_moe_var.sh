cd $GRAFT_REPO_ROOT
for i in 1 2 3; do timeout 600 python bench.py --model alexnet_moe --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/mv_$i.json 2> gpurun_out/mv_$i.err; done
python scripts/moe_e2e_probe.py > gpurun_out/mv_probe.log 2>&1
