#!/usr/bin/env bash
# Round-2 closing pass: GPU tests, smoke, bench, launch list and full ncu
# captures of the bench's kernels (tools/gpu_check_r2.sh), plus full captures
# of the FMNIST- and IMDb-shaped training kernels. The .ncu-rep files are
# summarised on the box (tools/summarize_ncu.py) and removed, so the merged
# gpurun_out/ stays under gpurun's 64 MiB.
tag=${1:-r2w}
bash tools/gpu_check_r2.sh $tag
for k in fmnist imdb; do
  TMG_KIND=$k timeout 600 ncu --set full --clock-control none --import-source on -k regex:train_async -c 1 \
    -o gpurun_out/prof_${k}_$tag -f python tools/variant_time.py 0 > gpurun_out/ncu_${k}_$tag.txt 2>&1
done
python tools/summarize_ncu.py gpurun_out/prof_train_$tag.ncu-rep gpurun_out/sum_train_async_$tag "" "profiles/${tag}_train_async.md (ncu --set full --clock-control none, bench.py MNIST fresh epoch)" > /dev/null
python tools/summarize_ncu.py gpurun_out/prof_evalb_$tag.ncu-rep gpurun_out/sum_eval_bits_$tag "" "profiles/${tag}_eval_bits.md (ncu --set full --clock-control none, bench.py inference)" > /dev/null
python tools/summarize_ncu.py gpurun_out/prof_fmnist_$tag.ncu-rep gpurun_out/sum_fmnist_async_$tag "" "profiles/${tag}_fmnist_async.md (ncu --set full, tools/variant_time.py FMNIST-shaped fresh epoch)" > /dev/null
python tools/summarize_ncu.py gpurun_out/prof_imdb_$tag.ncu-rep gpurun_out/sum_imdb_smem_$tag "" "profiles/${tag}_imdb_smem.md (ncu --set full, tools/variant_time.py IMDb-shaped fresh epoch)" > /dev/null
rm -f gpurun_out/*.ncu-rep
ls -la gpurun_out | tail -30
echo final-done
