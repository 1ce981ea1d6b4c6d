timeout 600 python -m pytest tests/test_gpu_generic.py tests/test_gpu_multirank.py tests/test_multirank_ipc.py tests/test_gpu_fd.py -x -q > gpurun_out/t12.log 2>&1; echo rc=$? >> gpurun_out/t12.log
timeout 300 python -m pytest tests/test_gpu_scale.py -x -q -k "c4 or rc" >> gpurun_out/t12.log 2>&1; echo rc=$? >> gpurun_out/t12.log
timeout 300 python bench.py --config c4w --no-cpu-baseline --no-e2e > gpurun_out/b12.log 2>&1
