cd $GRAFT_REPO_ROOT
nvidia-smi -L > gpurun_out/g1_smi.txt 2>&1
timeout 400 python -m pytest tests/test_gpu_ops.py -m gpu -q -k "not conv and not inner_product" > gpurun_out/g1_elem.log 2>&1
echo "elem rc=$?" >> gpurun_out/g1_elem.log
timeout 400 python -m pytest tests/test_gpu_ops.py -m gpu -q -k "inner_product" > gpurun_out/g1_ip.log 2>&1
echo "ip rc=$?" >> gpurun_out/g1_ip.log
timeout 600 python -m pytest tests/test_gpu_ops.py -m gpu -q -k "conv" > gpurun_out/g1_conv.log 2>&1
echo "conv rc=$?" >> gpurun_out/g1_conv.log
