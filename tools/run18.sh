timeout 900 python -m pytest tests/test_gpu_partition.py tests/test_gpu_scale.py tests/test_gpu_multirank.py tests/test_gpu_graph.py tests/test_ref_suites.py tests/test_gpu_engine.py tests/test_cpp.py tests/test_dumps.py tests/test_harness.py -x -q > gpurun_out/t18.log 2>&1; echo rc=$? >> gpurun_out/t18.log
timeout 300 python bench.py --partitions 8 --no-cpu-baseline --no-e2e > gpurun_out/b18.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-e2e >> gpurun_out/b18.log 2>&1
