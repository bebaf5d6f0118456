mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rA --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu_r1i.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_r1i.txt
timeout 300 python tools/variant_time.py 3 > gpurun_out/time_r1i.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:train_async -s 1 -c 1 -o gpurun_out/prof_train_r1i -f python tools/variant_time.py 1 > gpurun_out/ncu_r1i.txt 2>&1
timeout 900 python tools/sweep.py all > gpurun_out/sweep_r1i.jsonl 2> gpurun_out/sweep_r1i.err
echo done
