#!/usr/bin/env bash
# Persistent shared-memory clause kernel A/B (TMG_SMEM_PERSIST=0: launched
# CTAs) on the IMDb-shaped fresh epoch, after the wide-row tests.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "wide or smem or very_wide or imdb or shard" > gpurun_out/persist_pytest.txt 2>&1; echo "exit $?" >> gpurun_out/persist_pytest.txt; tail -n 2 gpurun_out/persist_pytest.txt
for v in 1 0 1 0; do
  TMG_SMEM_PERSIST=$v TMG_KIND=imdb timeout 600 python tools/variant_time.py 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('persist=$v', round(d['epoch0_ms'],1), d['epoch0_ms_all'], int(d['events']), d['acc_after_e1'])"
done
