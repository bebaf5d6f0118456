"""A scripted `tm` command-line session (the reference CLI surface,
proj/src/cli.cpp:429-530) and its normalised transcript: every command's exit
code and stdout, plus digests of the files it wrote (models, report and bench
CSVs, binarizer specs, synthetic datasets). Wall-clock seconds are masked;
everything else must match the reference byte for byte.

The same session runs against oracle/_ref/tm_ref (our CLI source linked with
the reference library; transcript committed as tests/golden/cli_session_ref.txt
by tests/gen_golden.sh) and against paper_2009_04861_b200/_lib/tm (the GPU
facade). Part "host" needs no GPU (synth, parse errors, missing files);
part "gpu" trains, evaluates and benches.

    python -m tests.cli_session <binary> [host|gpu|all]
"""
import hashlib
import os
import re
import subprocess
import sys
import tempfile

CSV_TEXT = (
    "temp,humidity,wind,rain,label\n"
    + "".join(
        f"{(i * 37) % 41 - 5.5},{(i * 13) % 97 / 7.0},{i % 3},{(i * 7) % 2},{(i * 5 + (i * 37) % 41) % 3}\n"
        for i in range(240)
    )
)

HOST = [
    ["synth", "--name", "xor", "--train", "64", "--test", "16", "--noise", "0.1", "--seed", "3", "--out", "xor"],
    ["synth", "--name", "patterns", "--train", "300", "--test", "100", "--classes", "3", "--zone", "4",
     "--noise", "0.05", "--seed", "5", "--out", "pat"],
    ["synth", "--name", "staircase", "--train", "200", "--test", "60", "--synth-features", "5", "--seed", "2",
     "--out", "stair"],
    ["synth", "--name", "spiral", "--out", "bad"],
    ["synth", "--out", "x"],
    [],
    ["fit"],
    ["train", "--bogus"],
    ["train", "--mode", "fast"],
    ["train", "--task", "cluster"],
    ["train", "--clauses", "ten"],
    ["train", "--seed", "-1"],
    ["train", "--clauses", "3", "--synth", "xor"],
    ["train", "--states", "0", "--synth", "xor"],
    ["train", "--data", "missing.txt"],
    ["train", "--synth", "xor", "--test", "pat.test"],
    ["train"],
    ["eval", "--data", "pat.test"],
    ["eval", "--model", "missing.txt", "--data", "pat.test"],
    ["bench", "--synth", "xor", "--bench-mode", "seq"],
    ["bench", "--clauses", "4", "--bench-mode", "sometimes"],
    ["train", "--epochs", "3", "--help"],
]

GPU = [
    ["train", "--synth", "patterns", "--synth-train", "300", "--synth-test", "100", "--classes", "3",
     "--zone", "4", "--clauses", "20", "--margin", "8", "--specificity", "3.5", "--epochs", "3", "--seed", "7",
     "--per-epoch", "--report", "seq.csv", "--out", "seq.model"],
    ["train", "--data", "pat.train", "--test", "pat.test", "--clauses", "12", "--epochs", "2", "--mode", "par",
     "--workers", "1", "--boost", "--states", "64", "--report", "par1.csv", "--out", "par1.model"],
    ["eval", "--model", "seq.model", "--data", "pat.test"],
    ["eval", "--model", "par1.model", "--data", "pat.train"],
    ["train", "--task", "regress", "--synth", "staircase", "--synth-train", "200", "--synth-test", "60",
     "--synth-features", "5", "--clauses", "16", "--margin", "10", "--epochs", "3", "--per-epoch",
     "--report", "reg.csv", "--out", "reg.model"],
    ["eval", "--model", "reg.model", "--data", "stair.test"],
    ["train", "--task", "regress", "--data", "stair.train", "--test", "stair.test", "--mode", "par",
     "--workers", "1", "--clauses", "10", "--epochs", "2", "--out", "regpar.model"],
    ["train", "--data", "w.csv", "--binarize-bits", "3", "--train-fraction", "0.75", "--clauses", "10",
     "--epochs", "2", "--binarizer-out", "w.bin", "--out", "w.model", "--report", "w.csv.report"],
    ["eval", "--model", "w.model", "--data", "w.csv", "--binarizer", "w.bin"],
    ["eval", "--model", "w.model", "--data", "w.csv"],
    ["train", "--task", "regress", "--data", "w.csv", "--binarize-bits", "2", "--clauses", "8", "--epochs", "2",
     "--out", "wreg.model"],
    ["train", "--synth", "xor", "--binarizer-out", "x.bin", "--epochs", "1", "--clauses", "4"],
    ["bench", "--synth", "patterns", "--synth-train", "120", "--synth-test", "40", "--clauses", "4,10",
     "--workers", "1", "--warmup", "1", "--bench-epochs", "2", "--seed", "9", "--out", "bench.csv"],
    ["bench", "--synth", "staircase", "--task", "regress", "--clauses", "6", "--bench-mode", "par",
     "--workers", "1", "--bench-epochs", "1"],
    ["bench", "--data", "pat.train", "--clauses", "4"],
    # TM_THREADS=1 turns --workers 8 into the one-worker (bit-exact) schedule
    ["@TM_THREADS=1", "train", "--data", "pat.train", "--test", "pat.test", "--mode", "par", "--workers", "8",
     "--clauses", "10", "--epochs", "2", "--out", "env.model"],
    ["@TM_THREADS=zero", "train", "--synth", "xor", "--epochs", "1", "--clauses", "4"],
]

_SECONDS = re.compile(r"(seconds )\S+")


def _mask_line(line):
    line = _SECONDS.sub(r"\1*", line)
    parts = line.split(",")
    if len(parts) == 7 and parts[0] in ("seq", "par"):  # report / bench CSV row: mask the seconds column
        parts[4] = "*"
        line = ",".join(parts)
    return line


def _digest(path):
    with open(path, "rb") as f:
        data = f.read()
    if path.endswith(".csv") or path.endswith(".report"):
        data = "\n".join(_mask_line(l) for l in data.decode().splitlines()).encode()
    return hashlib.sha256(data).hexdigest()[:16]


def run(binary, part="all", workdir=None):
    """Run the session; returns the transcript lines."""
    out = []
    with tempfile.TemporaryDirectory() as tmp:
        cwd = workdir or tmp
        with open(os.path.join(cwd, "w.csv"), "w") as f:
            f.write(CSV_TEXT)
        cmds = (HOST if part in ("host", "all") else []) + (GPU if part in ("gpu", "all") else [])
        if part == "gpu":  # the gpu part reads the synthetic files the host part writes
            cmds = HOST[:3] + GPU
        for cmd in cmds:
            env = dict(os.environ)
            env.pop("TM_THREADS", None)
            # one-worker `--mode par` runs replay the reference schedule bit-exactly
            # (TMG_MODE_AUTO); the reference binary ignores the variable
            env["TSETLIN_DETERMINISTIC"] = "1"
            args = list(cmd)
            while args and args[0].startswith("@"):
                k, v = args.pop(0)[1:].split("=", 1)
                env[k] = v
            before = set(os.listdir(cwd))
            p = subprocess.run([os.path.abspath(binary)] + args, cwd=cwd, env=env, capture_output=True, text=True, timeout=600)
            out.append("$ tm " + " ".join(cmd))
            out.append(f"rc {p.returncode}")
            out.extend(_mask_line(l) for l in p.stdout.splitlines())
            # error text (usage lines excluded): the first stderr line
            err = [l for l in p.stderr.splitlines() if l.strip()]
            if err and p.returncode in (1, 2):
                out.append("stderr " + err[0])
            for name in sorted(set(os.listdir(cwd)) - before):
                out.append(f"file {name} {_digest(os.path.join(cwd, name))}")
    return out


if __name__ == "__main__":
    print("\n".join(run(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "all")))
