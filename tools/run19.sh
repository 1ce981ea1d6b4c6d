timeout 600 python -m pytest tests/test_gpu_graph.py tests/test_gpu_generic.py tests/test_gpu_multirank.py tests/test_gpu_errors.py -x -q > gpurun_out/t19.log 2>&1; echo rc=$? >> gpurun_out/t19.log
timeout 300 python bench.py --config c4w --no-cpu-baseline --no-e2e > gpurun_out/b19.log 2>&1
