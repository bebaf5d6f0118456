# Clause-order experiment (TrainParams::interleave): accuracy (5 seeds) and
# fresh-epoch time at the MNIST, FMNIST and IMDb shapes for each order.
for o in class warp block; do
  TMG_CLAUSE_ORDER=$o python tools/acc_sched.py 3 $o
  for k in mnist fmnist imdb; do TMG_KIND=$k TMG_CLAUSE_ORDER=$o python tools/variant_time.py 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$o', d['kind'], round(d['epoch0_ms'],2), d['events'], round(d['acc_after_e0'],4), round(d['acc_after_e1'],4))"; done
done
