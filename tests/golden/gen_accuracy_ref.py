#!/usr/bin/env python3
"""Reference accuracy numbers for the asynchronous-training parity gate
(BASELINE.json: <=0.5 pt vs the reference, mean over 5 seeds).

Runs the UNMODIFIED reference (oracle/_ref/ref_driver, built by
oracle/Makefile from /root/reference) with train_epoch_parallel on all host
threads and records test accuracy per epoch into accuracy_ref.json.
"""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
DRIVER = os.path.join(HERE, "..", "..", "oracle", "_ref", "ref_driver")

CASES = {
    "xor_noise10": dict(data="xor", q=5000, qtest=5000, clauses=20, T=15, s=3.9, epochs=50,
                        noise=0.1, data_seed=7),
    "xor_noise40": dict(data="xor", q=5000, qtest=5000, clauses=20, T=15, s=3.9, epochs=50,
                        noise=0.4, data_seed=7),
    "xor_noise40_w1": dict(data="xor", q=5000, qtest=5000, clauses=20, T=15, s=3.9, epochs=50,
                           noise=0.4, data_seed=7, workers=1),
    "mnist_q6000": dict(data="mnist", q=6000, qtest=2000, clauses=2000, T=50, s=10.0, epochs=3,
                        noise=0.0, data_seed=2009),
    # BASELINE.json configs[2] / [3] shapes at the full clause counts, on a
    # training prefix the reference finishes in minutes.
    "fmnist_q1000": dict(data="fmnist", q=1000, qtest=2000, clauses=8000, T=100, s=15.0, epochs=2,
                         noise=0.0, data_seed=2352),
    "imdb_q4000": dict(data="imdb", q=4000, qtest=2000, clauses=10000, T=100, s=15.0, epochs=2,
                       noise=0.0, data_seed=10000),
    "mnist_q6000_w1": dict(data="mnist", q=6000, qtest=2000, clauses=2000, T=50, s=10.0, epochs=3,
                           noise=0.0, data_seed=2009, workers=1),
    # configs[2] / [3] shapes on larger training prefixes (about an hour of
    # the reference each on the 8-core build container)
    "fmnist_q6000": dict(data="fmnist", q=6000, qtest=2000, clauses=8000, T=100, s=15.0, epochs=2,
                         noise=0.0, data_seed=2352),
    "imdb_q12000": dict(data="imdb", q=12000, qtest=4000, clauses=10000, T=100, s=15.0, epochs=2,
                        noise=0.0, data_seed=10000),
    # the reference's own one-worker schedule at the IMDb shape (the band)
    "imdb_q4000_w1": dict(data="imdb", q=4000, qtest=2000, clauses=10000, T=100, s=15.0, epochs=2,
                          noise=0.0, data_seed=10000, workers=1, seeds=3),
    "imdb_q12000_w1": dict(data="imdb", q=12000, qtest=4000, clauses=10000, T=100, s=15.0, epochs=2,
                           noise=0.0, data_seed=10000, workers=1, seeds=1),
    # The configuration bench.py times (BASELINE.json configs[1]) at its full
    # size: q = 60 000 training rows, 10 000 test rows, 3 epochs.
    "mnist_q60000": dict(data="mnist", q=60000, qtest=10000, clauses=2000, T=50, s=10.0, epochs=3,
                         noise=0.0, data_seed=2009),
    # The reference's own worker-count spread at that configuration.
    "mnist_q60000_w1": dict(data="mnist", q=60000, qtest=10000, clauses=2000, T=50, s=10.0, epochs=3,
                            noise=0.0, data_seed=2009, workers=1, seeds=3),
    "mnist_q60000_w2": dict(data="mnist", q=60000, qtest=10000, clauses=2000, T=50, s=10.0, epochs=3,
                            noise=0.0, data_seed=2009, workers=2, seeds=3),
    "mnist_q60000_w4": dict(data="mnist", q=60000, qtest=10000, clauses=2000, T=50, s=10.0, epochs=3,
                            noise=0.0, data_seed=2009, workers=4, seeds=3),
}


def run(case, seed, workers):
    workers = case.get("workers", workers)
    args = [DRIVER, "train", "--data", case["data"], "--q", str(case["q"]), "--qtest", str(case["qtest"]),
            "--clauses", str(case["clauses"]), "--T", str(case["T"]), "--s", str(case["s"]),
            "--epochs", str(case["epochs"]), "--noise", str(case["noise"]), "--seed", str(seed),
            "--data-seed", str(case["data_seed"]), "--workers", str(workers)]
    out = subprocess.run(args, check=True, capture_output=True, text=True).stdout
    return [json.loads(l) for l in out.splitlines() if l.strip()]


def _update(path, name, fn):
    """Read-modify-write of accuracy_ref.json under an exclusive file lock
    (several generator processes may run at once)."""
    import fcntl
    with open(path + ".lock", "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        res = json.load(open(path)) if os.path.exists(path) else {}
        res[name] = fn(res.get(name))
        json.dump(res, open(path, "w"), indent=1)


def main():
    """Usage: gen_accuracy_ref.py [case ...]. Seeds already recorded for a case
    are kept (resume); the missing ones up to the case's seed count run in
    parallel when PARALLEL_SEEDS=1 (one-worker cases: one core each)."""
    from concurrent.futures import ThreadPoolExecutor
    names = sys.argv[1:] or list(CASES)
    path = os.path.join(HERE, "accuracy_ref.json")
    workers = os.cpu_count() or 1
    for name in names:
        case = CASES[name]
        old = (json.load(open(path)) if os.path.exists(path) else {}).get(name) or {}
        done = set(old.get("per_seed", {})) if old.get("config") == case or "seeds" in case else set()
        todo = [s for s in range(1, case.get("seeds", 5) + 1) if str(s) not in done]

        def one(seed):
            rows = run(case, seed, workers)
            acc = [r["test_accuracy"] for r in rows]
            print(name, seed, acc, [r["seconds"] for r in rows], flush=True)

            def merge(prev):
                prev = prev if prev and prev.get("per_seed") else {}
                per_seed = dict(prev.get("per_seed", {}))
                seconds = dict(prev.get("epoch_seconds", {}))
                events = dict(prev.get("feedback_events", {}))
                per_seed[str(seed)] = acc
                seconds[str(seed)] = [r["seconds"] for r in rows]
                events[str(seed)] = [r["feedback_events"] for r in rows]
                final = [v[-1] for v in per_seed.values()]
                return dict(config=case, workers=case.get("workers", workers), per_seed=per_seed,
                            mean_final=sum(final) / len(final), epoch_seconds=seconds, feedback_events=events)
            _update(path, name, merge)

        if os.environ.get("PARALLEL_SEEDS") == "1":
            with ThreadPoolExecutor(len(todo) or 1) as ex:
                list(ex.map(one, todo))
        else:
            for seed in todo:
                one(seed)


if __name__ == "__main__":
    main()
