"""Helpers to read the reference golden fixtures (tests/golden/, made by
tests/golden/gen_golden.sh from the compiled reference)."""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(*parts):
    return np.load(os.path.join(GOLDEN, *parts))


def manifest(*parts):
    with open(os.path.join(GOLDEN, *parts, "manifest.json")) as f:
        return json.load(f)


EPOCH_CASES = ["xor12", "mnist_small", "boost_n5"]
