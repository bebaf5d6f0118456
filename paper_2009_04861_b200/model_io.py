"""tmmodel v1 text model files (reference: proj/src/model_io.cpp:27-184;
SURVEY.md §8(f) row f3), byte-identical to the reference writer so trained
machines interchange with the CPU reference in both directions.

Only configuration and automaton counters are stored (model_io.cpp:35-57);
tallies, previous outputs, epoch and RNG state are not, exactly like the
reference.
"""
from __future__ import annotations

import numpy as np

from .tsetlin import MultiClassTM, RegressionHead, TMConfig


def _fmt(v: float) -> str:
    return "%.17g" % v  # format_double, model_io.cpp:29-33


def _config_lines(cfg: TMConfig) -> list:
    return [f"clauses {cfg.clauses}", f"margin {cfg.margin}", f"specificity {_fmt(cfg.specificity)}",
            f"states {cfg.state_depth}", f"boost {1 if cfg.boost_true_positive else 0}", f"seed {cfg.seed}"]


def _bank_lines(counters: np.ndarray, index: int) -> list:
    lines = [f"bank {index}"]
    lines += [" ".join(str(int(v)) for v in row) for row in counters]
    return lines


def dumps(model) -> str:
    """save_model (model_io.cpp:107-128) for a MultiClassTM or RegressionHead."""
    if isinstance(model, RegressionHead):
        lines = ["tmmodel v1", "task regress", f"features {model.feature_count()}",
                 f"range {_fmt(model.y_min)} {_fmt(model.y_max)}"] + _config_lines(model.config)
        lines += _bank_lines(model.bank.counters(), 0)
    else:
        lines = ["tmmodel v1", "task classify", f"features {model.feature_count()}",
                 f"classes {model.num_banks()}"] + _config_lines(model.config)
        for c in range(model.num_banks()):
            lines += _bank_lines(model.banks[c].counters(), c)
    return "\n".join(lines) + "\nend\n"


def save_model_file(path: str, model) -> None:
    with open(path, "w") as f:
        f.write(dumps(model))


class _Tokens:
    def __init__(self, text: str):
        self.tok, self.k = text.split(), 0

    def next(self) -> str:
        if self.k >= len(self.tok):
            raise RuntimeError("model parse: unexpected end of file")
        self.k += 1
        return self.tok[self.k - 1]

    def field(self, key: str, conv=int):
        k = self.next()
        v = self.next()
        if k != key:
            raise RuntimeError(f"model parse: expected '{key}' field")
        return conv(v)


def _read_config(t: _Tokens) -> TMConfig:  # model_io.cpp:75-87
    cfg = TMConfig()
    cfg.clauses = t.field("clauses")
    cfg.margin = t.field("margin")
    cfg.specificity = t.field("specificity", float)
    cfg.state_depth = t.field("states")
    cfg.boost_true_positive = t.field("boost") != 0
    cfg.seed = t.field("seed")
    cfg.epochs, cfg.workers = 0, 0
    return cfg


def _read_bank(t: _Tokens, index: int, n: int, L: int, N: int) -> np.ndarray:  # model_io.cpp:89-103
    if t.field("bank") != index:
        raise RuntimeError("model parse: bank index out of order")
    vals = np.empty(n * L, np.int64)
    for k in range(n * L):
        try:
            vals[k] = int(t.next())
        except RuntimeError:
            raise RuntimeError("model parse: truncated counter block")
        if vals[k] < 1 or vals[k] > 2 * N:
            raise RuntimeError(f"model parse: counter {vals[k]} outside [1, 2N]")
    return vals.reshape(n, L).astype(np.uint16)


def parse(text: str) -> dict:
    """Host-side parse of a tmmodel v1 text (model_io.cpp:130-165):
    {task, features, classes, config, range, banks: [n x 2o uint16]}."""
    t = _Tokens(text)
    if t.next() != "tmmodel" or t.next() != "v1":
        raise RuntimeError("model parse: not a tmmodel v1 file")
    task = t.field("task", str)
    out = {"task": task, "range": None}
    if task == "classify":
        out["features"], out["classes"] = t.field("features"), t.field("classes")
    elif task == "regress":
        out["features"], out["classes"] = t.field("features"), 1
        if t.next() != "range":
            raise RuntimeError("model parse: expected 'range' field")
        out["range"] = (float(t.next()), float(t.next()))
    else:
        raise RuntimeError(f"model parse: unknown task '{task}'")
    cfg = out["config"] = _read_config(t)
    out["banks"] = [_read_bank(t, c, cfg.clauses, 2 * out["features"], cfg.state_depth)
                    for c in range(out["classes"])]
    if t.next() != "end":
        raise RuntimeError("model parse: missing end marker")
    return out


def loads(text: str, device: int = 0):
    """load_model (model_io.cpp:130-165): MultiClassTM or RegressionHead on `device`."""
    p = parse(text)
    if p["task"] == "classify":
        tm = MultiClassTM(p["config"], p["features"], p["classes"], device=device)
        for c, counters in enumerate(p["banks"]):
            tm.banks[c].set_counters(counters)
        return tm
    head = RegressionHead(p["config"], p["features"], *p["range"], device=device)
    head.bank.set_counters(p["banks"][0])
    return head


def load_model_file(path: str, device: int = 0):
    with open(path) as f:
        return loads(f.read(), device)
