cd $GRAFT_REPO_ROOT
QNB_PATCH=1 timeout 900 ncu --set full --clock-control none --import-source on -k "regex:igemm_patch" -c 1 -o gpurun_out/ptprof3 \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --profile-reps 1 > gpurun_out/ptprof3_ncu.log 2>&1
