#!/usr/bin/env bash
# Fused saturating pass for rows of >= 2 words per lane: parity and timings.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "type_i_bit_exact or wide or fmnist or table1 or rates or invariants or golden or mirror or sequential or dropin or parity" > gpurun_out/satnw_pytest.txt 2>&1; echo "exit $?" >> gpurun_out/satnw_pytest.txt; tail -n 2 gpurun_out/satnw_pytest.txt
for k in fmnist mnist imdb; do
  TMG_KIND=$k timeout 600 python tools/variant_time.py 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$k', round(d['epoch0_ms'],1), [round(x,1) for x in d['epoch0_ms_all']], int(d['events']), d['acc_after_e1'])"
done
