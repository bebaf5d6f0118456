#!/usr/bin/env bash
# One gpurun call comparing build variants of libtmgpu.so on one dataset shape.
# Usage: bash tools/gpu_variants.sh <tag> <mnist|fmnist|imdb> ["name:EXTRA nvcc flags" ...]
# Writes gpurun_out/time_<tag>_<name>.json (plus _cur for the default build).
tag=$1; kind=$2; shift 2
mkdir -p gpurun_out
[ $# -gt 0 ] && bash tools/build_variants.sh "$@" > gpurun_out/variants_$tag.txt 2>&1
TMG_KIND=$kind timeout 300 python tools/variant_time.py ${REPS:-2} > gpurun_out/time_${tag}_cur.json 2>&1
for spec in "$@"; do
  name="${spec%%:*}"
  TMG_KIND=$kind TMG_LIB=$PWD/paper_2009_04861_b200/_lib/variants/$name/libtmgpu.so \
    timeout 300 python tools/variant_time.py ${REPS:-2} > gpurun_out/time_${tag}_$name.json 2>&1
done
echo done
