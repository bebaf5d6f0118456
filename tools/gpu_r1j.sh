mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_r1j.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -rA --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu_r1j.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_r1j.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r1j.txt 2>&1; echo "exit $?" >> gpurun_out/smoke_r1j.txt
timeout 300 python tools/variant_time.py 3 > gpurun_out/time_r1j.json 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r1j.json 2> gpurun_out/bench_r1j.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_r1j.json 2> gpurun_out/bench_ref_r1j.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_r1j.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch_r1j.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:train_async -s 1 -c 1 -o gpurun_out/prof_train_r1j -f python tools/variant_time.py 1 > gpurun_out/ncu_r1j.txt 2>&1
timeout 900 python tools/sweep.py all > gpurun_out/sweep_r1j.jsonl 2> gpurun_out/sweep_r1j.err
echo done
