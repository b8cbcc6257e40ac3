"""Repeated un-instrumented solves of C3 (200 iterations) in one process:
wall / device time per solve, to expose per-solve graph (re)build costs.
python tools/c3_repeat.py [iters] [repeats]"""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2502_09502_b200 as eng
from paper_2502_09502_b200 import data

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 200
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
cd = data.make_config("C3", scale=1.0)
inst = eng.ProblemInstance(cd.X, cd.y, eng.LossKind(cd.loss), cd.k, cd.M, cd.lambda2, dtype=cd.dtype)
L = 58143.30059520633
o = lambda k: eng.FistaOptions(lipschitz=L, max_iterations=k, gap_tolerance=1e-300, stop_on_gap=False)
eng.solve_relaxation(inst, opts=o(5), return_device=True)
torch.cuda.synchronize()
for i in range(reps):
    t0 = time.perf_counter()
    r = eng.solve_relaxation(inst, opts=o(iters), return_device=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"solve {i}: {dt*1e3:.1f} ms  {iters/dt:.1f} it/s  launches {r.stats['gpu_launches']} "
          f"full_prox {r.stats['prox_full_passes']} restarts {r.restarts}", flush=True)
