"""C4 (batched node relaxations) throughput: n=20000, p=5000 fp32, 512 nodes,
500 iterations each; prints node-iterations/s and the contraction's share."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2502_09502_b200 import (FistaOptions, LossKind, NodeState, ProblemInstance,
                                   solve_relaxation_batched)
from paper_2502_09502_b200.data import make_config

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
count = int(sys.argv[2]) if len(sys.argv) > 2 else 512
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 500
t0 = time.time()
cfg = make_config("C4", scale=scale, nodes=count)
inst = ProblemInstance(cfg.X, cfg.y, LossKind.SQUARED_ERROR, cfg.k, cfg.M, cfg.lambda2, dtype="fp32")
nodes = [None] + [NodeState(fixed_one=f1, fixed_zero=f0) for f0, f1 in cfg.nodes[:count - 1]]
print(f"gen {time.time()-t0:.1f}s", flush=True)
Xd = torch.from_numpy(cfg.X).cuda().double()
v = torch.randn(Xd.shape[1], device="cuda", dtype=torch.float64)
for _ in range(100):                       # power iteration on X^T X (model.py:283-306)
    w = Xd.T @ (Xd @ v)
    lam = float(w.norm())
    v = w / lam
L = 2.0 * 1.01 * lam
del Xd
opts = FistaOptions(max_iterations=iters, stop_on_gap=False, lipschitz=L)
solve_relaxation_batched(inst, nodes, opts=FistaOptions(max_iterations=3, stop_on_gap=False, lipschitz=L))
torch.cuda.synchronize()
t0 = time.time()
reps = solve_relaxation_batched(inst, nodes, opts=opts)
dt = time.time() - t0
print(f"C4 scale={scale} nodes={count} iters={iters}: {dt*1e3:.1f} ms  "
      f"{count*iters/dt:.0f} node-it/s  {dt/iters*1e3:.3f} ms/batched-iteration", flush=True)
print("gaps", np.percentile([r.gap for r in reps], [0, 50, 100]), "restarts",
      np.mean([r.restarts for r in reps]))

if __import__("os").environ.get("L0_DEBUG"):
    solve_relaxation_batched(inst, nodes, opts=FistaOptions(max_iterations=iters, stop_on_gap=False,
                                                            lipschitz=L, profile=True))
