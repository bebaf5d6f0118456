mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rA --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu_r1g.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_r1g.txt
timeout 600 python tools/calib_synth.py > gpurun_out/calib_r1g.jsonl 2> gpurun_out/calib_r1g.err
timeout 600 python tools/sweep.py imdb > gpurun_out/sweep_imdb_r1g.jsonl 2> gpurun_out/sweep_imdb_r1g.err
echo done
