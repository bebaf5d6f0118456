mkdir -p gpurun_out
bash tools/build_variants.sh "nolsb:-DTMG_SAMPLER_LSB=0" "nop2:-DTMG_ASYNC_P2=0" "minb6:-DTMG_ASYNC_MINB=6" "minb4:-DTMG_ASYNC_MINB=4" "minb8:-DTMG_ASYNC_MINB=8" > gpurun_out/variants_r1l.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu_r1l.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_r1l.txt
timeout 300 python tools/variant_time.py 3 > gpurun_out/time_r1l_cur.json 2>&1
for v in nolsb nop2 minb6 minb4 minb8; do
TMG_LIB=$PWD/paper_2009_04861_b200/_lib/variants/$v/libtmgpu.so timeout 300 python tools/variant_time.py 3 > gpurun_out/time_r1l_$v.json 2>&1
done
echo done
