mkdir -p gpurun_out
for v in minb0 minb5 minb6 minb8 minb6p7; do
  TMG_LIB=paper_2009_04861_b200/_lib/variants/$v/libtmgpu.so timeout 300 python tools/variant_time.py 3 >> gpurun_out/variants_r1c.jsonl 2>>gpurun_out/variants_r1c.err
done
echo done
