mkdir -p gpurun_out
bash tools/build_variants.sh "msb:-DTMG_SAMPLER_UBR=0" "msb8:-DTMG_SAMPLER_UBR=0 -DTMG_ASYNC_MINB=8" "msb6:-DTMG_SAMPLER_UBR=0 -DTMG_ASYNC_MINB=6" "ubr8:-DTMG_ASYNC_MINB=8" "ubr6:-DTMG_ASYNC_MINB=6" > gpurun_out/variants_r1m.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_async.py -q -x --timeout 600 -p no:cacheprovider -k bit_exact > gpurun_out/pytest_gpu_r1m.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_r1m.txt
timeout 300 python tools/variant_time.py 3 > gpurun_out/time_r1m_cur.json 2>&1
for v in msb msb8 msb6 ubr8 ubr6; do
TMG_LIB=$PWD/paper_2009_04861_b200/_lib/variants/$v/libtmgpu.so timeout 300 python tools/variant_time.py 3 > gpurun_out/time_r1m_$v.json 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:train_async -s 1 -c 1 -o gpurun_out/prof_train_r1m -f python tools/variant_time.py 1 > gpurun_out/ncu_r1m.txt 2>&1
echo done
