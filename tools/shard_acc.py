import sys, numpy as np
sys.path.insert(0, '.')
import paper_2009_04861_b200 as T
from paper_2009_04861_b200 import synth
d = synth.make("mnist", 6000, 2000, 2009)
for n in (400, 2000):
    for devs in (None, [0, 0], [0, 0, 0, 0]):
        cfg = T.TMConfig(clauses=n, margin=50, specificity=10.0, seed=42)
        tm = T.MultiClassTM(cfg, 784, 10, devices=devs)
        pool = T.ExamplePool(784, d.train_x, d.train_y, 10)
        test = T.ExamplePool(784, d.test_x, d.test_y, 10)
        out = []
        for e in range(3):
            rep = T.train_epoch_parallel(tm, pool, 8, e)
            out.append((rep.total_feedback_events(), round(T.evaluate_accuracy(tm, test), 4)))
        print(n, devs, out, flush=True)
