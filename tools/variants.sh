# A/B the model-kernel variants: bash tools/variants.sh ["conv bwd" ...]
# (GMD_CONV_VARIANT / GMD_BWD_VARIANT), after the model + multirank GPU tests.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -k "model or multirank" -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
[ $# -eq 0 ] && set -- "0 0" "1 4"
for v in "$@"; do
  set -- $v
  GMD_CONV_VARIANT=$1 GMD_BWD_VARIANT=$2 timeout 300 python bench.py --steps 10 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench_$1_$2.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bench_$1_$2.log').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$1 $2', round(d['ms_per_step'],3), 'conv', k['conv'], 'bwd', k['bwd_edge'])"
done
grep -E "passed|failed|Error|assert" gpurun_out/gpu_tests.log | tail -8
