"""Instance ingest (reference data.py:36-317):
synthetic generation, text loaders, standardize, the instance file format."""

import numpy as np
import pytest

from paper_2502_09502_b200 import data
from paper_2502_09502_b200.errors import DataFormatError, InvalidInputError


def test_generate_synthetic_matches_generator():
    inst = data.generate_synthetic(data.SyntheticParams(n=40, p=12, k_true=3, seed=4))
    X, y, bt = data.synthetic(40, 12, 3, seed=4)
    assert np.array_equal(inst.X, X) and np.array_equal(inst.y, y) and np.array_equal(inst.beta_true, bt)
    assert inst.k == 3 and inst.M == data.DEFAULT_M and inst.lambda2 == data.DEFAULT_LAMBDA2
    cls = data.generate_synthetic(data.SyntheticParams(n=40, p=12, k_true=3, task="classification"))
    assert set(np.unique(cls.y)) <= {-1.0, 1.0} and cls.loss.value == "logistic"
    for bad in (dict(n=0, p=3, k_true=1), dict(n=3, p=3, k_true=4), dict(n=3, p=3, k_true=1, sigma=1.0),
                dict(n=3, p=3, k_true=1, snr=0.0), dict(n=3, p=3, k_true=1, task="x"),
                dict(n=3, p=3, k_true=1, snr_scale="x")):
        with pytest.raises(InvalidInputError):
            data.SyntheticParams(**bad)


def test_load_delimited_and_sparse(tmp_path):
    f = tmp_path / "d.csv"
    f.write_text("# comment\n1,2,3\n\n4 5 6\n")
    X, y = data.load_dataset(f)
    assert X.tolist() == [[1.0, 2.0], [4.0, 5.0]] and y.tolist() == [3.0, 6.0]
    X, y = data.load_dataset(f, label_column="first")
    assert X.tolist() == [[2.0, 3.0], [5.0, 6.0]] and y.tolist() == [1.0, 4.0]
    s = tmp_path / "s.txt"
    s.write_text("1 1:0.5 3:2\n-1 2:1\n")
    X, y = data.load_dataset(s, fmt="sparse")
    assert X.tolist() == [[0.5, 0.0, 2.0], [0.0, 1.0, 0.0]] and y.tolist() == [1.0, -1.0]
    X, _ = data.load_dataset(s, fmt="sparse", n_features=5)
    assert X.shape == (2, 5)
    with pytest.raises(DataFormatError):
        data.load_dataset(s, fmt="sparse", n_features=2)
    bad = tmp_path / "bad.csv"
    bad.write_text("1,2,3\n1,2\n")
    with pytest.raises(DataFormatError) as e:
        data.load_dataset(bad)
    assert e.value.line == 2
    bad.write_text("1 0:2\n")
    with pytest.raises(DataFormatError) as e:
        data.load_dataset(bad, fmt="sparse")
    assert e.value.line == 1
    empty = tmp_path / "e.csv"
    empty.write_text("# nothing\n")
    with pytest.raises(DataFormatError):
        data.load_dataset(empty)
    with pytest.raises(InvalidInputError):
        data.load_dataset(f, fmt="json")


def test_standardize_and_back_mapping():
    rng = np.random.default_rng(0)
    X = rng.standard_normal((30, 5)) * [1, 2, 3, 4, 5] + [1, 0, -2, 3, 0]
    X[:, 2] = 7.0                                    # constant column
    Xs, tr = data.standardize(X)
    assert tr.kept.tolist() == [0, 1, 3, 4] and tr.dropped.tolist() == [2]
    assert np.allclose(Xs.mean(axis=0), 0.0, atol=1e-14)
    assert np.allclose(np.linalg.norm(Xs, axis=0), 1.0)
    b_std = rng.standard_normal(4)
    beta, icpt = tr.map_coefficients(b_std)
    assert beta[2] == 0.0
    # predictions agree: Xs b_std == X beta + intercept
    assert np.allclose(Xs @ b_std, X @ beta + icpt)
    with pytest.raises(InvalidInputError):
        data.standardize(np.ones((5, 3)))


def test_instance_round_trip(tmp_path):
    inst = data.generate_synthetic(data.SyntheticParams(n=9, p=4, k_true=2, seed=1))
    f = tmp_path / "inst.txt"
    data.write_instance(f, inst)
    back = data.read_instance(f)
    assert np.array_equal(back.X, inst.X) and np.array_equal(back.y, inst.y)
    assert back.k == inst.k and back.M == inst.M and back.lambda2 == inst.lambda2
    assert back.loss is inst.loss and np.array_equal(back.beta_true, inst.beta_true)
    text = f.read_text().replace("n 9", "n 8")
    f.write_text(text)
    with pytest.raises(DataFormatError):
        data.read_instance(f)
