# ncu --set full (source-level) capture of one kernel of the AlexNet INT8 bench forward.
# usage: gpu_ncu_kernel.sh TAG REGEX [extra env]
cd $GRAFT_REPO_ROOT
TAG=$1; K=$2
O=gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$K" -c 1 -o $O/${TAG} python bench.py --steps 1 --warmup 1 --no-cpu-baseline --profile-reps 1 > $O/${TAG}.log 2>&1
ncu -i $O/${TAG}.ncu-rep --page source --csv --print-source sass > $O/${TAG}_sass.csv 2>/dev/null
ncu -i $O/${TAG}.ncu-rep --page details > $O/${TAG}_details.txt 2>/dev/null
ncu -i $O/${TAG}.ncu-rep --page raw --csv > $O/${TAG}_raw.csv 2>/dev/null
rm -f $O/${TAG}.ncu-rep
