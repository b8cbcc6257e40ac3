import sys, time
sys.path.insert(0, ".")
import torch
import paper_2502_09502_b200.fista as F
from paper_2502_09502_b200 import (FistaOptions, LossKind, NodeState, ProblemInstance, lipschitz_constant)
from paper_2502_09502_b200.data import make_config
cfg = make_config("C4", scale=1.0, nodes=512)
inst = ProblemInstance(cfg.X, cfg.y, LossKind.SQUARED_ERROR, cfg.k, cfg.M, cfg.lambda2, dtype="fp32")
nodes = [None] + [NodeState(fixed_one=f1, fixed_zero=f0) for f0, f1 in cfg.nodes[:511]]
L = lipschitz_constant(inst, method="lanczos")
o = FistaOptions(max_iterations=1, stop_on_gap=False, lipschitz=L, gap_tolerance=1e-300)
F.solve_relaxation_batched(inst, nodes, opts=o, return_device=True)
torch.cuda.synchronize()
lib = F.native.load()
orig = lib.l0_batch_solve
def timed(*a):
    t0 = time.perf_counter(); r = orig(*a); print(f"   l0_batch_solve {1e3*(time.perf_counter()-t0):.2f} ms"); return r
class W:
    def __getattr__(self, k): return timed if k == "l0_batch_solve" else getattr(lib, k)
F.native.load = lambda: W()
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    F.solve_relaxation_batched(inst, nodes, opts=o, return_device=True)
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"solve {1e3*(t1-t0):.2f} ms (+sync {1e3*(t2-t1):.2f})")
t0 = time.perf_counter(); ps = [F.EnvelopeParams.for_instance(inst, nd) for nd in nodes]; print(f"params {1e3*(time.perf_counter()-t0):.2f} ms")
t0 = time.perf_counter(); dp = inst.device_problem(); h = dp.batch(len(nodes)); print(f"dp.batch {1e3*(time.perf_counter()-t0):.2f} ms")
