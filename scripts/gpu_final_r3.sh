# Round-2 (session 3) verification pass: full GPU tests, smoke, every bench line, the reference arm,
# ncu launch list + one --set full forward capture (with the tcgen05 UMMA counters).
cd $GRAFT_REPO_ROOT
TAG=${1:-r3z}
O=gpurun_out
UM=sm__ops_path_tensor_op_utcimma_src_int8_realtime.avg.pct_of_peak_sustained_elapsed,sm__ops_path_tensor_op_utcimma_src_int8_realtime.sum
timeout 1800 python -m pytest tests -m gpu -q -x -p no:hypothesispytest > $O/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> $O/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1
echo "smoke rc=$?" >> $O/${TAG}_smoke.log
timeout 600 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
timeout 600 python bench.py --impl reference > $O/${TAG}_ref.json 2> $O/${TAG}_ref.err
timeout 600 python bench.py --precision fp16 > $O/${TAG}_fp16.json 2> $O/${TAG}_fp16.err
timeout 600 python bench.py --precision int16 > $O/${TAG}_int16.json 2> $O/${TAG}_int16.err
timeout 900 python bench.py --model alexnet_moe --steps 30 --warmup 5 > $O/${TAG}_moe.json 2> $O/${TAG}_moe.err
timeout 900 python bench.py --model vgg16 --batch 128 --steps 10 --warmup 3 --no-cpu-baseline > $O/${TAG}_vgg.json 2> $O/${TAG}_vgg.err
timeout 1500 python bench.py --model convsweep --batch 128 --no-cpu-baseline > $O/${TAG}_sweep.json 2> $O/${TAG}_sweep.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --profile-reps 1 > /dev/null 2> $O/${TAG}_ncu.err
timeout 900 ncu --set full --metrics $UM --clock-control none --import-source on -k "regex:igemm|pack|pool|softmax|front" -c 14 -o $O/${TAG}_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline --profile-reps 1 > $O/${TAG}_full_ncu.log 2>&1
ncu -i $O/${TAG}_full.ncu-rep --page raw --csv > $O/${TAG}_full_raw.csv 2>/dev/null
ncu -i $O/${TAG}_full.ncu-rep --page details > $O/${TAG}_full_details.txt 2>/dev/null
rm -f $O/${TAG}_full.ncu-rep
bash scripts/gpu_ncu_kernel.sh ${TAG}_front front_kernel
rm -f $O/${TAG}_front_sass.csv.gz; gzip -f $O/${TAG}_front_sass.csv
