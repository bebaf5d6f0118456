# Round-2 measurement pass: full check (tests, smoke, bench, ncu), inference
# timings at three shapes, W=1 comparison, clause sweep with the reference.
set -u
bash tools/gpu_check_r2.sh r2h
timeout 900 python tools/eval_bench.py > gpurun_out/eval_r2h.jsonl 2> gpurun_out/eval_r2h.err
timeout 900 python tools/w1_compare.py 200 200 1000 2000 > gpurun_out/w1_r2h.jsonl 2> gpurun_out/w1_r2h.err
timeout 1800 python tools/sweep.py all 60000 --ref > gpurun_out/sweep_r2h.jsonl 2> gpurun_out/sweep_r2h.err
echo all-done
