#!/bin/bash
# One `ncu --set full` capture (with source) per "config:kernel" argument:
#   bash tools/ncu_one.sh TAG c4w:k_wide_bwd_edge_ff c5:k_nl_search ...
# (skips the first 3 launches of the kernel: warm-up steps)
T=$1; shift
mkdir -p gpurun_out
for ck in "$@"; do
  c=${ck%%:*}; k=${ck#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${k}\b" -s ${SKIP:-3} -c 1 \
      -o gpurun_out/${T}_${c}_${k} -f python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
      > gpurun_out/${T}_${c}_${k}.log 2>&1
  echo "$ck rc=$?"
done
