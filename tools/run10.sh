timeout 900 python -m pytest tests/test_gpu_graph.py tests/test_gpu_partition.py tests/test_gpu_scale.py tests/test_ref_suites.py -x -q > gpurun_out/t10.log 2>&1; echo rc=$? >> gpurun_out/t10.log
for c in c5 c4 c3; do timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e; done > gpurun_out/b10.log 2>&1
