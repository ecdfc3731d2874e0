# Profiles of the current code: launch list, one --set full forward (+ tcgen05 UMMA counters),
# and source-level SASS captures of conv1 (row-Hankel) and conv2 (CTA pair).
cd $GRAFT_REPO_ROOT
TAG=${1:-r2k}
O=gpurun_out
UM=sm__ops_path_tensor_op_utcimma_src_int8_realtime.avg.pct_of_peak_sustained_elapsed,sm__ops_path_tensor_op_utcimma_src_int8_realtime.sum
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --profile-reps 1 > /dev/null 2> $O/${TAG}_ncu.err
timeout 900 ncu --set full --metrics $UM --clock-control none --import-source on -k "regex:igemm|pack|pool|softmax" -c 16 -o $O/${TAG}_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline --profile-reps 1 > $O/${TAG}_full_ncu.log 2>&1
ncu -i $O/${TAG}_full.ncu-rep --page raw --csv > $O/${TAG}_full_raw.csv 2>/dev/null
ncu -i $O/${TAG}_full.ncu-rep --page details > $O/${TAG}_full_details.txt 2>/dev/null
rm -f $O/${TAG}_full.ncu-rep
for K in igemm_hk igemm_pair; do
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$K" -c 1 -o $O/${TAG}_$K python bench.py --steps 1 --warmup 1 --no-cpu-baseline --profile-reps 1 > $O/${TAG}_$K.log 2>&1
  ncu -i $O/${TAG}_$K.ncu-rep --page source --csv --print-source sass > $O/${TAG}_${K}_sass.csv 2>/dev/null
  ncu -i $O/${TAG}_$K.ncu-rep --page details > $O/${TAG}_${K}_details.txt 2>/dev/null
  rm -f $O/${TAG}_$K.ncu-rep
done
