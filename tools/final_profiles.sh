#!/bin/bash
# The round's committed profiles (run under gpurun): launch lists and ncu
# --set full captures of the hot kernels of C5, C4, C4w and the C5 p = 8
# partition kernels, then smoke() and the reference arm once.  Summarise
# with profiles/ncu_summary.py here.
R=${1:-r02c}
bash tools/profile_round.sh $R c5
KERNELS="k_bwd_edge2 k_conv2 k_tb_backward k_tb_forward" bash tools/profile_round.sh $R c4
KERNELS="k_wide_bwd_edge_sm k_wide_conv k_wide_tb_forward k_wide_node_tc" bash tools/profile_round.sh $R c4w
TAG=c5p8 EXTRA="--partitions 8 --no-e2e --no-cpu-baseline" \
    KERNELS="k_edge_lsrc k_lay_scatter k_lay_count k_sel_pass k_from_src k_owner" bash tools/profile_round.sh $R c5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${R}_refarm.log 2>&1; echo "ref rc=$?"
