timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t17.log 2>&1; echo rc=$? >> gpurun_out/t17.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke17.log 2>&1; echo rc=$? >> gpurun_out/smoke17.log
timeout 600 python bench.py > gpurun_out/b17_c5.log 2>&1
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/b17_ref.log 2>&1
for c in c4 c4w c3; do timeout 300 python bench.py --config $c; done > gpurun_out/b17_other.log 2>&1
GMD_BENCH_SHARE_GPU=1 timeout 300 python bench.py --gpus 2 --no-cpu-baseline > gpurun_out/b17_share2.log 2>&1
