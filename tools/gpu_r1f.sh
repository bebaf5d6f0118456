mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rA --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu_r1f.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_r1f.txt
timeout 900 python tools/sweep.py all > gpurun_out/sweep_r1f.jsonl 2> gpurun_out/sweep_r1f.err
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r1f.json 2> gpurun_out/bench_r1f.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_r1f.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch_r1f.txt 2>&1
echo done
