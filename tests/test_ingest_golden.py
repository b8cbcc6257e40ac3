"""Instance ingest against the reference's own outputs (SURVEY.md §8(f) rank
3): tests/golden/ingest.npz holds l0cert.data.load_dataset (data.py:122-201)
on the committed text files under tests/golden/ingest/ and
l0cert.data.standardize / map_coefficients (data.py:204-242) on seeded
matrices (tests/golden/make_golden_ingest.py).  Host paths are bit-exact; the
device standardize (CUDA tensors, csrc/standardize.cu) is bit-exact too."""

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
    """The device branch (csrc/standardize.cu) sums columns in numpy's order:
    bit-identical, including the wide-dynamic-range case whose centring
    cancels ~7 digits."""
    import torch
    X = torch.from_numpy(G[f"std{i}_in"]).cuda()
    out, tr = data.standardize(X)
    assert isinstance(out, torch.Tensor) and out.is_cuda
    assert np.array_equal(out.cpu().numpy(), G[f"std{i}_out"])
    assert np.array_equal(tr.kept, G[f"std{i}_kept"]) and np.array_equal(tr.dropped, G[f"std{i}_dropped"])
    assert np.array_equal(tr.means, G[f"std{i}_means"]) and np.array_equal(tr.norms, G[f"std{i}_norms"])
    beta, icpt = tr.map_coefficients(G[f"std{i}_bstd"])
    assert np.array_equal(beta, G[f"std{i}_beta"]) and icpt == float(G[f"std{i}_icpt"])


@pytest.mark.gpu
def test_standardize_device_fp32_and_errors():
    import torch
    X = G["std4_in"].astype(np.float32)
    out, tr = data.standardize(torch.from_numpy(X).cuda())
    ref, rtr = data.standardize(X)
    assert np.array_equal(out.cpu().numpy(), ref) and np.array_equal(tr.kept, rtr.kept)
    with pytest.raises(data.InvalidInputError):
        data.standardize(torch.ones((5, 3), dtype=torch.float64, device="cuda"))
    with pytest.raises(data.InvalidInputError):
        data.standardize(torch.ones((1, 3), dtype=torch.float64, device="cuda"))
