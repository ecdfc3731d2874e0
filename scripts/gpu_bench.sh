cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/b1.json 2> gpurun_out/b1.err
echo "bench rc=$?" >> gpurun_out/b1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/b1_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --profile-reps 1 > /dev/null 2> gpurun_out/b1_ncu.err
echo "ncu rc=$?" >> gpurun_out/b1_ncu.err
