"""Lanczos recurrence of spectral.py on the CPU (torch CPU tensors, no
engine): against LAPACK at 1e-12, and row-sharded over two gloo ranks (the
all-reduced X^T X v of ShardedProblem.lipschitz(method="lanczos"))."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")


def _op(X):
    Xt = torch.from_numpy(X)
    return lambda v: Xt.T @ (Xt @ v)


@pytest.mark.parametrize("n,p,rho", [(400, 300, 0.5), (1000, 200, 0.9), (150, 400, 0.0)])
def test_lanczos_cpu_matches_lapack(n, p, rho):
    from paper_2502_09502_b200.data import ar1_rows
    from paper_2502_09502_b200.spectral import lanczos_lambda_max
    X = ar1_rows(n, p, rho, np.random.default_rng(n + p))
    lam_ref = float(np.linalg.eigvalsh(X.T @ X)[-1])
    lam = lanczos_lambda_max(_op(X), p, "cpu")
    assert lam == pytest.approx(lam_ref, rel=1e-12)


def test_lanczos_rank_one_invariant_subspace():
    from paper_2502_09502_b200.spectral import lanczos_lambda_max
    a = np.random.default_rng(0).standard_normal(64)
    X = np.outer(np.ones(10), a)                # rank one: lambda = 10 ||a||^2
    lam = lanczos_lambda_max(_op(X), 64, "cpu")
    assert lam == pytest.approx(10.0 * float(a @ a), rel=1e-12)


def _worker(rank, world, port, X, out):
    import torch.distributed as dist
    from paper_2502_09502_b200.spectral import lanczos_lambda_max
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = X.shape[0]
    r0, r1 = rank * n // world, (rank + 1) * n // world
    lam = lanczos_lambda_max(_op(np.ascontiguousarray(X[r0:r1])), X.shape[1], "cpu",
                             allreduce=lambda t: dist.all_reduce(t))
    out[rank] = lam
    dist.destroy_process_group()


def test_lanczos_row_sharded_gloo():
    import multiprocessing as mp
    from paper_2502_09502_b200.data import ar1_rows
    X = ar1_rows(600, 250, 0.7, np.random.default_rng(5))
    lam_ref = float(np.linalg.eigvalsh(X.T @ X)[-1])
    ctx = mp.get_context("spawn")
    with ctx.Manager() as m:
        out = m.dict()
        port = 29500 + os.getpid() % 1000
        ps = [ctx.Process(target=_worker, args=(r, 2, port, X, out)) for r in range(2)]
        for p_ in ps:
            p_.start()
        for p_ in ps:
            p_.join(120)
            assert p_.exitcode == 0
        assert out[0] == out[1]                 # every rank runs the same recurrence
        assert out[0] == pytest.approx(lam_ref, rel=1e-12)
