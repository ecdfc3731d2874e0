# ncu --set full of one kernel (regex $2, $3 launches) in a short bench run
cd $GRAFT_REPO_ROOT
TAG=${1:-k}
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$2" -c ${3:-1} -o gpurun_out/${TAG} \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --profile-reps 1 > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${TAG}_ncu.log
