#!/usr/bin/env bash
# compute-sanitizer memcheck + racecheck over the deterministic replays
# (sequential trainer, grid and one-CTA; W = 1 mirror with jump-ahead draws)
# and the wide-row async kernels (x-only rows, packed last slot, persistent
# shared-memory kernel).
# Usage (under gpurun): bash tools/sanitize_seq.sh [tag]
tag="${1:-r2}"
mkdir -p gpurun_out
for tool in memcheck racecheck; do
  timeout 2400 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 --target-processes all \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_dropin.py tests/test_gpu_async.py -q -x -p no:cacheprovider \
    -k "sequential_parallel_replay or w1_replay_jump or sequential_trainer_bit_exact or sync_mirror_epochs or (wide and not accuracy) or smem or type_i_bit_exact" \
    > gpurun_out/sanitize_${tool}_$tag.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitize_${tool}_$tag.txt
  tail -3 gpurun_out/sanitize_${tool}_$tag.txt
done
