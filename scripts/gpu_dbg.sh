cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/dbg_tests.log 2>&1
echo "rc=$?" >> gpurun_out/dbg_tests.log
timeout 900 ncu --set full --clock-control none -k "regex:igemm" --launch-skip 5 -c 6 -o gpurun_out/p3 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --profile-reps 1 > gpurun_out/p3_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/p3_ncu.log
