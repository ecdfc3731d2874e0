# Round-2 measurement pass: tcgen05 MMA ceiling (+ ncu validation of the UMMA op counter),
# new GPU tests, conv sweep (configs[4]), AlexNet FP16 / INT16 lines, per-kernel UMMA utilisation.
cd $GRAFT_REPO_ROOT
TAG=${1:-r2b}
O=gpurun_out
timeout 120 scripts/_bin/int8_peak > $O/${TAG}_peak.json 2> $O/${TAG}_peak.err
M=gpu__time_duration.sum,sm__ops_path_tensor_op_utcimma_src_int8_realtime.sum,sm__ops_path_tensor_op_utcimma_src_int8_realtime.avg.pct_of_peak_sustained_elapsed,sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32_realtime.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tc.sum
timeout 300 ncu --metrics $M --clock-control none --csv scripts/_bin/int8_peak 20000 > $O/${TAG}_peak_ncu.csv 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -p no:hypothesispytest -k "batch256 or moe_gate or depth_bound or model_store or executor" > $O/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> $O/${TAG}_tests.log
timeout 1500 python bench.py --model convsweep --batch 128 --no-cpu-baseline > $O/${TAG}_sweep.json 2> $O/${TAG}_sweep.err
timeout 600 python bench.py --precision fp16 > $O/${TAG}_fp16.json 2> $O/${TAG}_fp16.err
timeout 600 python bench.py --precision int16 > $O/${TAG}_int16.json 2> $O/${TAG}_int16.err
timeout 600 ncu --metrics $M --clock-control none --csv -k regex:igemm -c 8 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/${TAG}_umma_ncu.csv 2>&1
