# round-2 refresh: launch lists (c5, c4, c4w) + ncu --set full of the C4w kernels
for c in c5 c4 c4w; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b_launches_${c}.csv \
      python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02b_launches_${c}.log 2>&1
  echo "launches $c rc=$?"
done
SKIP=3 bash tools/ncu_one.sh r02b c4w:k_wide_bwd_edge_sm c4w:k_wide_conv c4w:k_wide_tb_forward c4w:k_wide_tb_back1 c4w:k_wide_tb_back2 c4w:k_wide_bwd_node c4w:k_wide_tb_t
GMD_WIDE_TC=1 SKIP=3 bash tools/ncu_one.sh r02tc c4w:k_wide_bwd_edge
