mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu_r1n.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_r1n.txt
timeout 300 python tools/variant_time.py 3 > gpurun_out/time_r1n.json 2>&1
timeout 900 python tools/sweep.py fmnist > gpurun_out/sweep_fmnist_r1n.jsonl 2>&1
timeout 900 python tools/sweep.py imdb > gpurun_out/sweep_imdb_r1n.jsonl 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r1n.json 2> gpurun_out/bench_r1n.err
echo done
