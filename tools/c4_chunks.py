"""C4 batched solve time vs graph chunk length (per-chunk host round trip)."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2502_09502_b200 as eng
from paper_2502_09502_b200.data import make_config
cfg = make_config("C4", scale=1.0, nodes=512)
inst = eng.ProblemInstance(cfg.X, cfg.y, eng.LossKind.SQUARED_ERROR, cfg.k, cfg.M, cfg.lambda2, dtype="fp32")
nodes = [None] + [eng.NodeState(fixed_one=f1, fixed_zero=f0) for f0, f1 in cfg.nodes[:511]]
L = eng.lipschitz_constant(inst, method="lanczos")
for G in (10, 10, 25, 50, 100):
    o = eng.FistaOptions(max_iterations=100, stop_on_gap=False, lipschitz=L, chunk_iterations=G)
    eng.solve_relaxation_batched(inst, nodes, opts=o, return_device=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eng.solve_relaxation_batched(inst, nodes, opts=o, return_device=True)
    e1.record(); torch.cuda.synchronize()
    print(f"G={G}: {e0.elapsed_time(e1):.2f} ms per 100-iteration solve", flush=True)
