"""Where the e2e C2 solve (host numpy X -> solve to rel. gap 1e-6) spends its
time: upload + problem setup (device_problem) vs the solve itself.
python tools/e2e_breakdown.py"""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2502_09502_b200 as eng
from paper_2502_09502_b200 import data

cd = data.make_config("C2", scale=1.0)
L = 2.9908e5
for i in range(4):
    inst = eng.ProblemInstance(cd.X, cd.y, eng.LossKind.SQUARED_ERROR, cd.k, cd.M, cd.lambda2)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    inst.device_problem()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    r = eng.solve_relaxation(inst, opts=eng.FistaOptions(lipschitz=L, gap_tolerance=1e-300, gap_tolerance_rel=1e-6))
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    r2 = eng.solve_relaxation(inst, opts=eng.FistaOptions(lipschitz=L, gap_tolerance=1e-300, gap_tolerance_rel=1e-6))
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"device_problem {1e3*(t1-t0):.1f} ms, first solve {1e3*(t2-t1):.1f} ms ({r.iterations} its), "
          f"second solve same problem {1e3*(t3-t2):.1f} ms", flush=True)
    inst.release_device()
