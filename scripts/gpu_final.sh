# Round-end style pass: full GPU tests, smoke, bench (alexnet, moe, vgg), reference arm,
# ncu launch list + one --set full capture of the whole AlexNet forward.
cd $GRAFT_REPO_ROOT
TAG=${1:-fin}
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --model alexnet_moe --steps 30 --warmup 5 > gpurun_out/${TAG}_moe.json 2> gpurun_out/${TAG}_moe.err
timeout 900 python bench.py --model vgg16 --batch 128 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_vgg.json 2> gpurun_out/${TAG}_vgg.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --profile-reps 1 > /dev/null 2> gpurun_out/${TAG}_ncu.err
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:igemm|pack|pool|softmax" -c 16 -o gpurun_out/${TAG}_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline --profile-reps 1 > gpurun_out/${TAG}_full_ncu.log 2>&1
# the report itself can exceed gpurun's 64 MiB copy-back limit: keep its exports only
ncu -i gpurun_out/${TAG}_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_full_raw.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_full.ncu-rep --page details > gpurun_out/${TAG}_full_details.txt 2>/dev/null
rm -f gpurun_out/${TAG}_full.ncu-rep
