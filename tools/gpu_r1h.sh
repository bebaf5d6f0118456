mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rA --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu_r1h.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_r1h.txt
timeout 600 python tools/calib_synth.py > gpurun_out/calib_r1h.jsonl 2> gpurun_out/calib_r1h.err
echo done
