timeout 600 python -m pytest tests/test_gpu_model.py tests/test_gpu_physics.py tests/test_gpu_multirank.py tests/test_multirank_ipc.py tests/test_gpu_fd.py tests/test_ref_suites.py -x -q > gpurun_out/t14.log 2>&1; echo rc=$? >> gpurun_out/t14.log
timeout 300 python -m pytest tests/test_gpu_scale.py -x -q -k "c4 or rc" >> gpurun_out/t14.log 2>&1; echo rc=$? >> gpurun_out/t14.log
timeout 300 python bench.py --config c4 --no-cpu-baseline --no-e2e > gpurun_out/b14.log 2>&1
