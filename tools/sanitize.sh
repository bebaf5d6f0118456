#!/usr/bin/env bash
# compute-sanitizer memcheck + racecheck over small GPU cases (SURVEY.md §5:
# race freedom by construction, checked). Usage (under gpurun): bash tools/sanitize.sh [tag]
tag="${1:-r1}"
mkdir -p gpurun_out
for tool in memcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python -m pytest tests/test_gpu_async.py tests/test_gpu_parity.py -q -x -p no:cacheprovider \
    -k "bit_exact or invariants or window or contended or golden or random_states or margin" \
    > gpurun_out/sanitize_${tool}_$tag.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitize_${tool}_$tag.txt
done
