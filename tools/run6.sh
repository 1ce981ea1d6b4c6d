timeout 600 python -m pytest tests/test_gpu_fd.py tests/test_gpu_generic.py tests/test_gpu_multirank.py -x -q -s > gpurun_out/t6.log 2>&1; echo rc=$? >> gpurun_out/t6.log
timeout 300 python bench.py --config c4w --no-cpu-baseline --no-e2e > gpurun_out/b6.log 2>&1
bash tools/ncu_one.sh p3 c5:k_bwd_edge2 c5:k_conv2
