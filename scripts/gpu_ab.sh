# A/B of env knobs on the default AlexNet INT8 bench line: gpu_ab.sh TAG "ENV1" "ENV2" ...
cd $GRAFT_REPO_ROOT
TAG=$1; shift
i=0
for E in "" "$@"; do
  env $E timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/${TAG}_$i.json 2>/dev/null
  echo "$i $E" >> gpurun_out/${TAG}_index.txt
  i=$((i+1))
done
