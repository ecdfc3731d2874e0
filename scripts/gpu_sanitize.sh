cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none -k "regex:igemm_pair" -c 2 -o gpurun_out/pairchk python bench.py --steps 1 --warmup 1 --no-cpu-baseline --profile-reps 1 > gpurun_out/pairchk.log 2>&1
echo "ncu rc=$?" >> gpurun_out/pairchk.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -c "
import sys; sys.path.insert(0, '.')
import torch, bench
class A: model='alexnet'; precision='int8'; batch=8; steps=1; warmup=1
wl = bench.Workload(A, 0, 1)
wl.step(); torch.cuda.synchronize(); print('memcheck forward ok')
" > gpurun_out/memcheck.log 2>&1
echo "memcheck rc=$?" >> gpurun_out/memcheck.log
