set -x
timeout 600 python -m pytest tests/test_gpu_generic.py tests/test_gpu_physics.py tests/test_gpu_multirank.py -x -q > gpurun_out/t2.log 2>&1; echo rc=$? >> gpurun_out/t2.log
timeout 300 python -m pytest tests/test_gpu_scale.py -x -q -k c4 > gpurun_out/t2s.log 2>&1; echo rc=$? >> gpurun_out/t2s.log
for v in "" "GMD_WIDE_FF=16" "GMD_WIDE_TC=1"; do echo "== $v"; env $v timeout 300 python bench.py --config c4w --no-cpu-baseline --no-e2e; done > gpurun_out/b2.log 2>&1
