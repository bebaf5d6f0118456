#!/usr/bin/env bash
# Jump-ahead segment count (TMG_JUMP_SEGMENTS) A/B: the W = 1 replay and the
# sequential replay, MNIST- and IMDb-shaped, after the replay parity tests.
# (TMG_JUMP_SEGMENTS was an experiment knob in engine.cu jump_chunk, removed after this A/B: 32 segments stay.)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "sequential or mirror or w1 or jump or dropin or golden" > gpurun_out/seg_pytest.txt 2>&1; echo "exit $?" >> gpurun_out/seg_pytest.txt; tail -n 2 gpurun_out/seg_pytest.txt
TMG_JUMP_SEGMENTS=4 timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "sequential_parallel_replay or w1_replay_jump" 2>&1 | tail -n 1
for g in default 4 8 16 32; do
  if [ $g = default ]; then unset TMG_JUMP_SEGMENTS; else export TMG_JUMP_SEGMENTS=$g; fi
  echo "segments=$g"
  timeout 300 python - <<'PY'
import json, os, sys, time
sys.path.insert(0, ".")
import paper_2009_04861_b200 as T
from paper_2009_04861_b200 import synth
out = {}
d = synth.make("mnist", 200, 4, 2009)
tm = T.MultiClassTM(T.TMConfig(clauses=200, margin=50, specificity=10.0, seed=42), 784, 10)
pool = T.ExamplePool(784, d.train_x, d.train_y, 10)
rep = T.train_epoch_parallel(tm, pool, 1, 0, mode=T.MODE_SYNC_MIRROR)
out["w1_mnist_q200_n200_s"] = rep.device_seconds
for kind, q, n, Tm, s, seed in (("mnist", 500, 2000, 50, 10.0, 2009), ("imdb", 100, 10000, 100, 15.0, 10000)):
    d = synth.make(kind, q, 10, seed)
    tm = T.MultiClassTM(T.TMConfig(clauses=n, margin=Tm, specificity=s, seed=42), d.features, d.classes)
    pool = T.ExamplePool(d.features, d.train_x, d.train_y, d.classes)
    t0 = time.perf_counter(); rep = T.train_epoch_sequential(tm, pool, 0)
    out[f"seq_{kind}_s"] = time.perf_counter() - t0
    out[f"seq_{kind}_events"] = rep.total_feedback_events()
print(json.dumps(out))
PY
done
