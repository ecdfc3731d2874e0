cd $GRAFT_REPO_ROOT
run() { tag=$1; shift; env "$@" timeout 400 ncu $NCUARGS -k "regex:igemm_pair" -c 1 --log-file gpurun_out/$tag.txt python bench.py --steps 1 --warmup 1 --no-cpu-baseline --profile-reps 1 > gpurun_out/$tag.log 2>&1; echo "$tag $* rc=$?"; }
NCUARGS="--section SpeedOfLight --clock-control none" run pd1
NCUARGS="--set full --clock-control none" run pd2 QNB_NO_RELU_FREE=1
NCUARGS="--set full --clock-control none" run pd3 QNB_NO_PAIR_STREAM=1
NCUARGS="--set full --clock-control none --replay-mode application" run pd4
