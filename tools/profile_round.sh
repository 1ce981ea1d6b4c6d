#!/bin/bash
# Profile one round's headline workload on the GPU box (run under gpurun):
#   bash tools/profile_round.sh r01 [config]
# 1. launch list of one timed bench step (ncu gpu__time_duration.sum, every
#    launch; cold-cache and serialised: compare SHARES, not absolutes);
# 2. one `ncu --set full` capture per hot kernel (first launch after warm-up).
# Outputs land in gpurun_out/; summarise here with profiles/ncu_summary.py.
set -u
R=${1:-r01}
C=${2:-c5}
T=${TAG:-$C}            # output tag (e.g. c5p8 with EXTRA="--partitions 8")
X=${EXTRA:-}            # extra bench.py arguments
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none \
    --csv --log-file gpurun_out/${R}_launches_${T}.csv \
    python bench.py --config $C $X --steps 1 --warmup 3 > gpurun_out/${R}_launches_${T}.log 2>&1
echo "launch list rc=$?"
for k in ${KERNELS:-k_bwd_edge2 k_conv2 k_nl_search k_nl_emit k_bwd_node}; do
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:${k} \
        -s 0 -c 1 -o gpurun_out/${R}_${T}_${k} -f \
        python bench.py --config $C $X --steps 1 --warmup 3 > gpurun_out/${R}_${T}_${k}.log 2>&1
    echo "$k rc=$?"
done
