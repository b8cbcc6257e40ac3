"""Multi-rank host logic of the row-/node-sharded engine, world_size 2 over
gloo on CPU.

The engine's row-sharded mode all-reduces exactly these quantities per
iteration: [X_r^T grad F(u_gamma,r) | X_r^T zeta_r | F*(-zeta) partial sums]
and the loss partial sum, then runs the prox / envelope / restart logic
redundantly on every rank.  ``sharded_fista`` below performs that
decomposition with numpy partials and gloo all-reduces and must reproduce the
single-process oracle; the device side of the same path is checked on one GPU
in tests/test_gpu_distributed.py (all-reduce elided).
"""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_09502_b200 import data as mydata
from paper_2502_09502_b200 import distributed as shard


def test_row_range_partitions_rows():
    for n in (1, 7, 16000, 1_000_003):
        for world in (1, 2, 3, 8):
            spans = [shard.row_range(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                assert a1 == b0
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_shard_nodes_round_robin():
    nodes = list(range(10))
    got = sorted(i for r in range(3) for i in shard.shard_nodes(nodes, 3, r))
    assert got == nodes
    assert shard.shard_nodes(nodes, 3, 1) == [1, 4, 7]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def sharded_fista(X, y, loss, k, M, lam2, L, iters, allreduce):
    """Row-sharded restarted FISTA with the engine's decomposition (numpy)."""
    from oracle import l0_oracle as o
    two = 2.0 * lam2
    rho = L / two
    p = X.shape[1]
    beta = np.zeros(p)
    beta_prev = beta.copy()
    u = X @ beta
    u_prev = u.copy()
    obj = allreduce(np.array([o.loss_value(loss, u, y)]))[0] + two * o.envelope(beta, k, M)
    phi, restarts = 1, 0
    best = -math.inf
    trace = []
    for t in range(1, iters + 1):
        c = phi / (phi + 3.0)
        u_g = u + c * (u - u_prev)                    # X gamma by linearity (local rows)
        grad = allreduce(X.T @ o.loss_grad(loss, u_g, y))
        gam = beta + c * (beta - beta_prev)
        gam = gam - grad / L
        nxt = gam - o.prox_conj(rho * gam, rho, k, M) / rho
        u_prev, u = u, X @ nxt
        obj_new = allreduce(np.array([o.loss_value(loss, u, y)]))[0] + two * o.envelope(nxt, k, M)
        restarted = obj_new >= obj
        phi, restarts = (1, restarts + 1) if restarted else (phi + 1, restarts)
        beta_prev, beta, obj = beta, nxt, obj_new
        if t == 1 or t % 10 == 0:
            zeta = -o.loss_grad(loss, u, y)
            if loss == "squared_error":
                parts = allreduce(np.array([zeta @ zeta, y @ zeta]))
                fstar = 0.25 * parts[0] - parts[1]
            else:
                fstar = o.loss_conj_neg(loss, zeta, y)  # test uses squared error only
            v = allreduce(X.T @ zeta)
            d = -fstar - two * o.envelope_conj(v / two, k, M)
            best = max(best, d)
            trace.append((t, obj, best))
    return beta, obj, best, restarts, trace


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import l0_oracle as o
        out = {}
        # id exchange
        payload = bytes(range(128)) if rank == 0 else None
        out["bytes"] = shard.broadcast_bytes(payload, src=0) == bytes(range(128))
        # problem rows
        cd = mydata.make_config("C2", scale=1 / 40)       # n = p = 400
        r0, r1 = shard.row_range(cd.n, world, rank)
        Xr, yr = cd.X[r0:r1], cd.y[r0:r1]
        red = shard._torch_allreduce()
        v0 = o.power_start(cd.p)
        lam, its = shard.power_iteration(lambda v: Xr @ v, lambda w: Xr.T @ w, red, v0,
                                         tol=1e-10, max_iter=5000)
        out["lam"] = lam
        L = 2.0 * 1.01 * lam
        beta, obj, best, restarts, trace = sharded_fista(Xr, yr, cd.loss, cd.k, cd.M, cd.lambda2,
                                                         L, 60, red)
        out.update(beta=beta, obj=obj, best=best, restarts=restarts, trace=trace, L=L)
        shard.assert_replicated(beta)
        out["replicated"] = True
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_row_sharded_decomposition(oracle):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p_ in procs:
        p_.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    r0, r1 = res[0], res[1]
    assert r0["bytes"] and r1["bytes"] and r0["replicated"]
    # both ranks hold bitwise-identical replicated state
    assert np.array_equal(r0["beta"], r1["beta"]) and r0["obj"] == r1["obj"]
    # and it is the single-process algorithm
    cd = mydata.make_config("C2", scale=1 / 40)
    lam = oracle.lambda_max_power(cd.X, tol=1e-10, max_iter=5000)
    assert r0["lam"] == pytest.approx(lam, rel=1e-9)
    ref = oracle.fista(cd.X, cd.y, cd.loss, cd.k, cd.M, cd.lambda2, L=r0["L"], max_iter=60,
                       gap_tol=1e-300)
    assert r0["obj"] == pytest.approx(ref["primal_value"], rel=1e-12)
    assert r0["best"] == pytest.approx(ref["dual_bound"], rel=1e-9)
    np.testing.assert_allclose(r0["beta"], ref["beta"], rtol=0, atol=1e-10)
