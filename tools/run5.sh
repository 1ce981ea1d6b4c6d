timeout 600 python -m pytest tests/test_gpu_fd.py -x -q -s > gpurun_out/t5.log 2>&1; echo rc=$? >> gpurun_out/t5.log
bash tools/ncu_one.sh p2 c4w:k_wide_tb_forward c4w:k_wide_tb_back1
