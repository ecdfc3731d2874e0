# One ncu --set full capture of the named kernels during a short bench run.
# usage: bash scripts/gpu_ncu.sh TAG "regex:pack_input|pool_lrn|igemm" COUNT
cd $GRAFT_REPO_ROOT
TAG=${1:-prof}
KRE=${2:-regex:igemm}
CNT=${3:-3}
timeout 900 ncu --set full --clock-control none --import-source on -k "$KRE" -c $CNT -o gpurun_out/${TAG} \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --profile-reps 1 > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${TAG}_ncu.log
