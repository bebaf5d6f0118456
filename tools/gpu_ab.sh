#!/usr/bin/env bash
# A/B timing of the default build against tools/build_variants.sh variants on
# the MNIST / FMNIST / IMDb-shaped fresh async epoch, after a parity subset.
# Usage: bash tools/gpu_ab.sh <tag> "<pytest -k expr>" variant ...
tag=$1; k=$2; shift 2
mkdir -p gpurun_out
if [ -n "$k" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "$k" > gpurun_out/ab_${tag}_pytest.txt 2>&1
  echo "pytest exit $?" >> gpurun_out/ab_${tag}_pytest.txt; tail -2 gpurun_out/ab_${tag}_pytest.txt
fi
for kind in ${KINDS:-mnist fmnist imdb}; do
  for v in cur "$@"; do
    if [ $v = cur ]; then L=; else L=$PWD/paper_2009_04861_b200/_lib/variants/$v/libtmgpu.so; fi
    TMG_KIND=$kind TMG_LIB=$L timeout 600 python tools/variant_time.py ${REPS:-2} >> gpurun_out/ab_${tag}.jsonl 2>> gpurun_out/ab_${tag}.err
  done
done
python - "$tag" <<'PY'
import json, sys
for l in open(f"gpurun_out/ab_{sys.argv[1]}.jsonl"):
    d = json.loads(l)
    print(d["kind"], d["lib"].split("/")[-2], round(d["epoch0_ms"], 1), int(d["events"]), round(d["acc_after_e1"], 4))
PY
