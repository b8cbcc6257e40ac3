"""Golden fixtures for instance ingest: the
reference's own ``l0cert.data.load_dataset`` (data.py:122-201) on seeded text
files and ``l0cert.data.standardize`` (data.py:224-242) on seeded matrices.

Run in the BUILD container only (imports the reference from /root/reference):

    python tests/golden/make_golden_ingest.py

Writes the text files under tests/golden/ingest/ and the reference outputs to
tests/golden/ingest.npz.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
from l0cert import data as rdata  # noqa: E402  (the reference)

DIR = os.path.join(HERE, "ingest")
OUT = {}


def fmt(v, rng):
    style = rng.integers(0, 3)
    return repr(float(v)) if style == 0 else (f"{v:.6g}" if style == 1 else f"{v:.17e}")


def write_delimited(name, n, p, sep, seed, comments=True):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, p)) * rng.uniform(0.1, 50, p)
    X[:, rng.integers(0, p)] = 3.25                       # a constant column
    y = rng.standard_normal(n)
    lines = ["# seeded fixture"] if comments else []
    for i in range(n):
        row = [fmt(v, rng) for v in X[i]] + [fmt(y[i], rng)]
        lines.append(sep.join(row))
        if comments and i % 7 == 3:
            lines.append("")
    with open(os.path.join(DIR, name), "w") as fh:
        fh.write("\n".join(lines) + "\n")


def write_sparse(name, n, p, seed):
    rng = np.random.default_rng(seed)
    lines = []
    for i in range(n):
        idx = np.sort(rng.choice(p, size=rng.integers(0, max(1, p // 2)), replace=False)) + 1
        toks = [f"{int(rng.choice([-1, 1]))}"] + [f"{j}:{fmt(rng.standard_normal(), rng)}" for j in idx]
        lines.append(" ".join(toks))
    with open(os.path.join(DIR, name), "w") as fh:
        fh.write("\n".join(lines) + "\n")


def main():
    os.makedirs(DIR, exist_ok=True)
    write_delimited("comma.csv", 37, 9, ",", 1)
    write_delimited("space.txt", 23, 5, " ", 2)
    write_delimited("tabs.txt", 11, 4, "\t", 3, comments=False)
    write_sparse("sparse.svm", 29, 13, 4)
    cases = [("comma.csv", "delimited", "last", None), ("comma.csv", "delimited", "first", None),
             ("space.txt", "delimited", "last", None), ("tabs.txt", "delimited", "first", None),
             ("sparse.svm", "sparse", "last", None), ("sparse.svm", "sparse", "last", 20)]
    for i, (f, fm, lab, nf) in enumerate(cases):
        X, y = rdata.load_dataset(os.path.join(DIR, f), fmt=fm, label_column=lab, n_features=nf)
        OUT[f"load{i}_X"], OUT[f"load{i}_y"] = X, y
    OUT["load_cases"] = np.array([f"{f}|{fm}|{lab}|{nf if nf else 0}" for f, fm, lab, nf in cases])
    # standardize on loaded data and on seeded matrices (constant columns, wide
    # dynamic range, integer-valued, one tall-skinny, one wide)
    mats = [OUT["load0_X"], OUT["load2_X"], OUT["load4_X"]]
    rng = np.random.default_rng(7)
    A = rng.standard_normal((200, 30)) * np.logspace(-6, 6, 30) + rng.uniform(-1e3, 1e3, 30)
    A[:, [3, 17]] = [1.5, -2.0]
    mats.append(A)
    mats.append(rng.integers(-5, 6, size=(64, 40)).astype(np.float64))
    mats.append(rng.standard_normal((800, 7)))
    mats.append(rng.standard_normal((9, 150)))
    for i, M in enumerate(mats):
        out, tr = rdata.standardize(M)
        OUT[f"std{i}_in"], OUT[f"std{i}_out"] = M, out
        OUT[f"std{i}_kept"], OUT[f"std{i}_dropped"] = tr.kept, tr.dropped
        OUT[f"std{i}_means"], OUT[f"std{i}_norms"] = tr.means, tr.norms
        b = rng.standard_normal(tr.kept.size)
        beta, icpt = tr.map_coefficients(b)
        OUT[f"std{i}_bstd"], OUT[f"std{i}_beta"], OUT[f"std{i}_icpt"] = b, beta, np.array(icpt)
    OUT["std_count"] = np.array(len(mats))
    np.savez_compressed(os.path.join(HERE, "ingest.npz"), **OUT)
    print("wrote", len(OUT), "arrays")


if __name__ == "__main__":
    main()
