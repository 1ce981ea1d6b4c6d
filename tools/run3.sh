timeout 600 python -m pytest tests/test_gpu_generic.py tests/test_gpu_physics.py tests/test_gpu_multirank.py -x -q > gpurun_out/t3.log 2>&1; echo rc=$? >> gpurun_out/t3.log
for v in sm sm8 ff; do echo "== $v"; GMD_WIDE_BWD=$v timeout 300 python bench.py --config c4w --no-cpu-baseline --no-e2e; done > gpurun_out/b3.log 2>&1
