"""Per-solve fixed cost of the batched engine on C4: device time of
solve_relaxation_batched for several iteration counts (slope = per batched
iteration, intercept = per solve).  python tools/c4_fixed.py"""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2502_09502_b200 import (FistaOptions, LossKind, NodeState, ProblemInstance,
                                   lipschitz_constant, solve_relaxation_batched)
from paper_2502_09502_b200.data import make_config

cfg = make_config("C4", scale=1.0, nodes=512)
inst = ProblemInstance(cfg.X, cfg.y, LossKind.SQUARED_ERROR, cfg.k, cfg.M, cfg.lambda2, dtype="fp32")
nodes = [None] + [NodeState(fixed_one=f1, fixed_zero=f0) for f0, f1 in cfg.nodes[:511]]
L = lipschitz_constant(inst, method="lanczos")
o = lambda k: FistaOptions(max_iterations=k, stop_on_gap=False, lipschitz=L, gap_tolerance=1e-300)
solve_relaxation_batched(inst, nodes, opts=o(3))
rows = []
for k in (1, 10, 50, 100, 200):
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        solve_relaxation_batched(inst, nodes, opts=o(k), return_device=True)
        e1.record()
        torch.cuda.synchronize()
        ts.append((e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3))
    d, w = np.median([t[0] for t in ts]), np.median([t[1] for t in ts])
    rows.append((k, d))
    print(f"K={k:4d} device {d:8.2f} ms wall {w:8.2f} ms per-it {d / k:.4f}", flush=True)
A = np.vstack([[r[0] for r in rows], np.ones(len(rows))]).T
slope, icpt = np.linalg.lstsq(A, np.array([r[1] for r in rows]), rcond=None)[0]
print(f"fit: {slope:.4f} ms per batched iteration + {icpt:.2f} ms per solve")
