"""Per-solve fixed cost on C2: device time (CUDA events) and host wall time of
solve_relaxation(max_iterations=K) for several K; the slope is the per-
iteration time, the intercept the fixed cost.  python tools/fixed_cost.py"""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2502_09502_b200 as eng
from paper_2502_09502_b200 import data

cd = data.make_config("C2", scale=float(sys.argv[1]) if len(sys.argv) > 1 else 1.0)
inst = eng.ProblemInstance(cd.X, cd.y, eng.LossKind.SQUARED_ERROR, cd.k, cd.M, cd.lambda2)
inst.device_problem()
L = 2.9908e5
o = lambda k: eng.FistaOptions(lipschitz=L, max_iterations=k, gap_tolerance=1e-300, stop_on_gap=False)
for k in (3, 20, 200):
    eng.solve_relaxation(inst, opts=o(k), return_device=True)
torch.cuda.synchronize()
rows = []
for k in (1, 2, 5, 10, 20, 50, 100, 200, 400):
    dev, wall = [], []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record()
        rep = eng.solve_relaxation(inst, opts=o(k), return_device=True)
        e1.record()
        torch.cuda.synchronize()
        wall.append((time.perf_counter() - t0) * 1e3)
        dev.append(e0.elapsed_time(e1))
    rows.append((k, float(np.median(dev)), float(np.median(wall)), rep.stats["gpu_launches"]))
    print(f"K={k:4d} device {rows[-1][1]:8.3f} ms  wall {rows[-1][2]:8.3f} ms  per-it {rows[-1][1]/k:.4f} ms  launches {rows[-1][3]}", flush=True)
ks = np.array([r[0] for r in rows], float)
ds = np.array([r[1] for r in rows])
A = np.vstack([ks, np.ones_like(ks)]).T
slope, icpt = np.linalg.lstsq(A, ds, rcond=None)[0]
print(f"fit: {slope:.4f} ms/iteration + {icpt:.3f} ms fixed per solve")
