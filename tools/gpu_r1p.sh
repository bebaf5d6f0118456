mkdir -p gpurun_out
bash tools/build_variants.sh "mb4:-DTMG_ASYNC_MINB=4" "mb5:-DTMG_ASYNC_MINB=5" "nop2:-DTMG_ASYNC_P2=0" "v4mb5:-DTMG_ASYNC_V5=0 -DTMG_ASYNC_MINB=5" > gpurun_out/variants_r1p.txt 2>&1
TMG_KIND=fmnist timeout 300 python tools/variant_time.py 1 > gpurun_out/time_r1p_fm_cur.json 2>&1
for v in mb4 mb5 nop2 v4mb5; do
TMG_KIND=fmnist TMG_LIB=$PWD/paper_2009_04861_b200/_lib/variants/$v/libtmgpu.so timeout 300 python tools/variant_time.py 1 > gpurun_out/time_r1p_fm_$v.json 2>&1
done
timeout 300 python tools/variant_time.py 2 > gpurun_out/time_r1p_mn_cur.json 2>&1
timeout 300 python tools/e2e_breakdown.py > gpurun_out/e2e_r1p.json 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu_r1p.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_r1p.txt
echo done
