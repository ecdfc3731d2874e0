# A/B of environment switches on the AlexNet INT8 bench: one bench line per setting.
cd $GRAFT_REPO_ROOT
TAG=${1:-ab}
shift
for setting in "$@"; do
  name=$(echo "$setting" | tr ' =' '__')
  env $setting timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_${name}.json 2> gpurun_out/${TAG}_${name}.err
done
