"""C2 iterations/s with and without the per-kernel profile events in the graphs."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2502_09502_b200 as eng
from paper_2502_09502_b200 import data
cd = data.make_config("C2", scale=1.0)
inst = eng.ProblemInstance(cd.X, cd.y, eng.LossKind.SQUARED_ERROR, cd.k, cd.M, cd.lambda2)
for prof in (False, True, False, True):
    o = lambda k: eng.FistaOptions(lipschitz=2.9908e5, max_iterations=k, gap_tolerance=1e-300,
                                   stop_on_gap=False, profile=prof)
    eng.solve_relaxation(inst, opts=o(5), return_device=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    r = eng.solve_relaxation(inst, opts=o(400), return_device=True)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    print(f"profile={prof}: {400 / ms * 1e3:.1f} it/s ({ms / 400 * 1e3:.1f} us/it)", flush=True)
