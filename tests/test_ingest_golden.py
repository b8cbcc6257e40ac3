"""Instance ingest against the reference's own outputs (SURVEY.md §8(f) rank
3): tests/golden/ingest.npz holds l0cert.data.load_dataset (data.py:122-201)
on the committed text files under tests/golden/ingest/ and
l0cert.data.standardize / map_coefficients (data.py:204-242) on seeded
matrices (tests/golden/make_golden_ingest.py).  Host paths are bit-exact; the
device standardize (CUDA tensors) agrees to 1e-12 relative (summation order)."""

import os

import numpy as np
import pytest

from paper_2502_09502_b200 import data

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "ingest.npz"))


def _load_cases():
    for i, spec in enumerate(G["load_cases"]):
        f, fm, lab, nf = str(spec).split("|")
        yield i, os.path.join(HERE, "golden", "ingest", f), fm, lab, (int(nf) or None)


@pytest.mark.parametrize("case", list(_load_cases()), ids=lambda c: str(c[0]))
def test_load_dataset_matches_reference(case):
    i, path, fm, lab, nf = case
    X, y = data.load_dataset(path, fmt=fm, label_column=lab, n_features=nf)
    assert np.array_equal(X, G[f"load{i}_X"]) and np.array_equal(y, G[f"load{i}_y"])


@pytest.mark.parametrize("i", range(int(G["std_count"])))
def test_standardize_host_matches_reference(i):
    out, tr = data.standardize(G[f"std{i}_in"])
    assert np.array_equal(out, G[f"std{i}_out"])
    assert np.array_equal(tr.kept, G[f"std{i}_kept"]) and np.array_equal(tr.dropped, G[f"std{i}_dropped"])
    assert np.array_equal(tr.means, G[f"std{i}_means"]) and np.array_equal(tr.norms, G[f"std{i}_norms"])
    beta, icpt = tr.map_coefficients(G[f"std{i}_bstd"])
    assert np.array_equal(beta, G[f"std{i}_beta"]) and icpt == float(G[f"std{i}_icpt"])


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(int(G["std_count"])))
def test_standardize_device_matches_reference(i):
    import torch
    X = torch.from_numpy(G[f"std{i}_in"]).cuda()
    out, tr = data.standardize(X)
    assert isinstance(out, torch.Tensor) and out.is_cuda
    ref = G[f"std{i}_out"]
    got = out.cpu().numpy()
    assert got.shape == ref.shape
    assert np.max(np.abs(got - ref)) <= 1e-12 * max(1.0, float(np.max(np.abs(ref))))
    assert np.array_equal(tr.kept, G[f"std{i}_kept"]) and np.array_equal(tr.dropped, G[f"std{i}_dropped"])
    for name in ("means", "norms"):
        r = G[f"std{i}_{name}"]
        assert np.allclose(getattr(tr, name), r, rtol=1e-12, atol=1e-12 * max(1.0, float(np.max(np.abs(r)))))
    beta, icpt = tr.map_coefficients(G[f"std{i}_bstd"])
    assert np.allclose(beta, G[f"std{i}_beta"], rtol=1e-11, atol=0)
    assert abs(icpt - float(G[f"std{i}_icpt"])) <= 1e-10 * max(1.0, abs(float(G[f"std{i}_icpt"])))
