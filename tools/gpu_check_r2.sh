#!/usr/bin/env bash
# One gpurun call: GPU tests, smoke, bench, ncu launch list + full captures of
# the training and inference kernels of the bench command.
# Usage (from the repo root, under gpurun): bash tools/gpu_check_r2.sh <tag>
set -u
tag="${1:-r2}"
out=gpurun_out
mkdir -p "$out"
nvidia-smi > "$out/nvidia_smi_$tag.txt" 2>&1
nproc > "$out/nproc_$tag.txt"
if [ "${TESTS:-1}" = "1" ]; then
  ( timeout 1500 python -m pytest tests -m gpu -q -rA --timeout 1200 -p no:cacheprovider ${PYTEST_ARGS:-} > "$out/pytest_gpu_$tag.txt" 2>&1; echo "exit $?" >> "$out/pytest_gpu_$tag.txt" )
  tail -3 "$out/pytest_gpu_$tag.txt"
  ( timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$out/smoke_$tag.txt" 2>&1; echo "exit $?" >> "$out/smoke_$tag.txt" )
fi
if [ "${BENCH:-1}" = "1" ]; then
  ( timeout 1200 python bench.py ${BENCH_ARGS:-} > "$out/bench_$tag.json" 2> "$out/bench_$tag.err"; echo "exit $?" >> "$out/bench_$tag.err" )
  tail -c 3000 "$out/bench_$tag.json"; tail -3 "$out/bench_$tag.err"
fi
if [ "${NCU:-1}" = "1" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv \
      --log-file "$out/launches_$tag.csv" python bench.py --steps 2 --warmup 3 --no-cpu --no-other-configs > "$out/ncu_launch_bench_$tag.txt" 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:train_async -s 1 -c 1 \
      -o "$out/prof_train_$tag" -f python bench.py --steps 1 --warmup 3 --no-cpu --no-other-configs > "$out/ncu_full_train_$tag.txt" 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:eval_bits -s 3 -c 1 \
      -o "$out/prof_evalb_$tag" -f python bench.py --steps 1 --warmup 3 --no-cpu --no-other-configs > "$out/ncu_full_eval_$tag.txt" 2>&1
fi
echo done
