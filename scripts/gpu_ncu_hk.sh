cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:igemm_hk" -c 1 -o gpurun_out/hk python bench.py --steps 1 --warmup 1 --no-cpu-baseline --profile-reps 1 > gpurun_out/hk.log 2>&1
ncu -i gpurun_out/hk.ncu-rep --page source --csv --print-source sass > gpurun_out/hk_sass.csv 2>/dev/null
ncu -i gpurun_out/hk.ncu-rep --page details > gpurun_out/hk_details.txt 2>/dev/null
ncu -i gpurun_out/hk.ncu-rep --page raw --csv > gpurun_out/hk_raw.csv 2>/dev/null
rm -f gpurun_out/hk.ncu-rep
