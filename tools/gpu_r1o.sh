mkdir -p gpurun_out
bash tools/build_variants.sh "mb3:-DTMG_ASYNC_MINB=3" "mb4:-DTMG_ASYNC_MINB=4" "mb5:-DTMG_ASYNC_MINB=5" "mb6:-DTMG_ASYNC_MINB=6" > gpurun_out/variants_r1o.txt 2>&1
for v in mb4 mb5 mb6; do
TMG_KIND=fmnist TMG_LIB=$PWD/paper_2009_04861_b200/_lib/variants/$v/libtmgpu.so timeout 300 python tools/variant_time.py 1 > gpurun_out/time_r1o_fm_$v.json 2>&1
done
TMG_KIND=fmnist timeout 300 python tools/variant_time.py 1 > gpurun_out/time_r1o_fm_cur.json 2>&1
timeout 300 python tools/e2e_breakdown.py > gpurun_out/e2e_r1o.json 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r1o.json 2> gpurun_out/bench_r1o.err
echo done
