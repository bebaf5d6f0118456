#!/usr/bin/env bash
# Packed last word slot (ClausePk) A/B on the FMNIST-shaped fresh epoch
# (TMG_ASYNC_PACK=0: the plain layout), after the Type I parity and the
# wide-row tests.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "type_i_bit_exact or wide or fmnist or table1 or rates or invariants or shard or dist" > gpurun_out/pack_pytest.txt 2>&1; echo "exit $?" >> gpurun_out/pack_pytest.txt; tail -n 2 gpurun_out/pack_pytest.txt
for v in 1 0 1 0; do
  TMG_ASYNC_PACK=$v TMG_KIND=fmnist timeout 600 python tools/variant_time.py 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pack=$v', round(d['epoch0_ms'],1), [round(x,1) for x in d['epoch0_ms_all']], int(d['events']), d['acc_after_e0'], d['acc_after_e1'])"
done
