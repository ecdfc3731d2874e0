# ncu --set full over one whole AlexNet INT8 forward (skips the weight-quantize launches
# of finalize_quantizers), plus the launch list.  usage: bash scripts/gpu_ncu_full.sh TAG
cd $GRAFT_REPO_ROOT
TAG=${1:-full}
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:igemm|pack|pool|softmax" -s 0 -c 15 \
  -o gpurun_out/${TAG} python bench.py --steps 1 --warmup 1 --no-cpu-baseline --profile-reps 1 > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${TAG}_ncu.log
