# ncu launch list + one --set full capture of one AlexNet INT8 forward.  usage: bash scripts/gpu_ncu_only.sh TAG
cd $GRAFT_REPO_ROOT
TAG=${1:-ncu}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --profile-reps 1 > /dev/null 2> gpurun_out/${TAG}_ncu.err
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:igemm|pack|pool|softmax" -c 16 -o gpurun_out/${TAG}_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline --profile-reps 1 > gpurun_out/${TAG}_full_ncu.log 2>&1
ncu -i gpurun_out/${TAG}_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_full_raw.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_full.ncu-rep --page details > gpurun_out/${TAG}_full_details.txt 2>/dev/null
ls -la gpurun_out/ > gpurun_out/${TAG}_ls.txt
rm -f gpurun_out/${TAG}_full.ncu-rep
