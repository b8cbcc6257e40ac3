"""Host -> HBM upload of a pageable numpy X (csrc/upload.cu l0_upload_rows:
multi-threaded pinned staging ring overlapped with the DMA; the drop-in
path of ProblemInstance with numpy X, model.py:75-116): bitwise copies for
ragged shapes (row blocks not a multiple of the staging slot, padded row
pitch ld > p with zero padding), fp64 and fp32 storage, and the device
cache keyed by the array object."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,p,dtype", [(1, 5, np.float64), (3001, 1001, np.float64),
                                       (70001, 300, np.float32), (257, 32, np.float64),
                                       (9000, 2048, np.float32)])
def test_upload_bitwise(engine, n, p, dtype):
    rng = np.random.default_rng(n + p)
    X = rng.standard_normal((n, p)).astype(dtype)
    y = rng.standard_normal(n)
    inst = engine.ProblemInstance(X, y, engine.LossKind.SQUARED_ERROR, 1, 1.0, 1.0,
                                  dtype="fp32" if dtype == np.float32 else "fp64")
    dp = inst.device_problem()
    Xd = dp.X.cpu().numpy()
    assert Xd.shape == (n, dp.ld) and dp.ld % 32 == 0 and dp.ld >= p
    assert np.array_equal(Xd[:, :p], X)
    assert not np.any(Xd[:, p:])


def test_device_cache_follows_the_array_object(engine):
    rng = np.random.default_rng(1)
    X = rng.standard_normal((50, 20))
    inst = engine.ProblemInstance(X, rng.standard_normal(50), engine.LossKind.SQUARED_ERROR, 2, 1.0, 1.0)
    d1 = inst.device_problem()
    assert inst.device_problem() is d1
    inst.X = X * 2.0                       # a new array: re-uploaded
    d2 = inst.device_problem()
    assert d2 is not d1 and np.array_equal(d2.X.cpu().numpy()[:, :20], X * 2.0)
