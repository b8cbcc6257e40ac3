"""Host-side cost of a batched C4 solve (512 nodes, 1 iteration): cProfile of
solve_relaxation_batched.  python tools/c4_host.py"""
import cProfile, pstats, sys, time
sys.path.insert(0, ".")
import torch
from paper_2502_09502_b200 import (FistaOptions, LossKind, NodeState, ProblemInstance,
                                   lipschitz_constant, solve_relaxation_batched)
from paper_2502_09502_b200.data import make_config

cfg = make_config("C4", scale=1.0, nodes=512)
inst = ProblemInstance(cfg.X, cfg.y, LossKind.SQUARED_ERROR, cfg.k, cfg.M, cfg.lambda2, dtype="fp32")
nodes = [None] + [NodeState(fixed_one=f1, fixed_zero=f0) for f0, f1 in cfg.nodes[:511]]
L = lipschitz_constant(inst, method="lanczos")
o = FistaOptions(max_iterations=1, stop_on_gap=False, lipschitz=L, gap_tolerance=1e-300)
solve_relaxation_batched(inst, nodes, opts=o, return_device=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
solve_relaxation_batched(inst, nodes, opts=o, return_device=True)
torch.cuda.synchronize()
print(f"one 1-iteration batched solve: {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
pr = cProfile.Profile()
pr.enable()
solve_relaxation_batched(inst, nodes, opts=o, return_device=True)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(14)
