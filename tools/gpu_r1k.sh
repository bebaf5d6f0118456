mkdir -p gpurun_out
bash tools/build_variants.sh "v4:-DTMG_ASYNC_V5=0" > gpurun_out/variants_r1k.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu_r1k.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_r1k.txt
timeout 300 python tools/variant_time.py 3 > gpurun_out/time_r1k_v5.json 2>&1
TMG_LIB=$PWD/paper_2009_04861_b200/_lib/variants/v4/libtmgpu.so timeout 300 python tools/variant_time.py 3 > gpurun_out/time_r1k_v4.json 2>&1
timeout 300 python tools/e2e_breakdown.py > gpurun_out/e2e_r1k.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:train_async -s 1 -c 1 -o gpurun_out/prof_train_r1k -f python tools/variant_time.py 1 > gpurun_out/ncu_r1k.txt 2>&1
echo done
