#!/usr/bin/env bash
# compute-sanitizer memcheck + racecheck over the round-2 kernels: the
# example-sliced class sums (list build, transpose, eval_bits, refresh) and the
# clause-sharded machines (replicas, windowed exchange, peer_sum_kernel).
# Usage (under gpurun): bash tools/sanitize_r2.sh [tag]
tag="${1:-r2}"
mkdir -p gpurun_out
for tool in memcheck racecheck; do
  timeout 2400 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 --target-processes all \
    python -m pytest tests/test_gpu_eval.py tests/test_gpu_shards.py tests/test_gpu_parity.py -q -x -p no:cacheprovider \
    -k "long_lists or range or python_api or one_rank or inference or refresh or update_clause or rebinds" \
    > gpurun_out/sanitize_${tool}_$tag.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitize_${tool}_$tag.txt
  tail -3 gpurun_out/sanitize_${tool}_$tag.txt
done
