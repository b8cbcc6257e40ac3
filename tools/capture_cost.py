"""Does the timed K-iteration solve pay a graph capture?  W-iteration warm-up
(as bench.py), then two K-iteration solves timed with CUDA events.
python tools/capture_cost.py [K] [W]"""
import sys
sys.path.insert(0, ".")
import torch
import paper_2502_09502_b200 as eng
from paper_2502_09502_b200 import data

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
W = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cd = data.make_config("C2", scale=1.0)
inst = eng.ProblemInstance(cd.X, cd.y, eng.LossKind.SQUARED_ERROR, cd.k, cd.M, cd.lambda2)
o = lambda k: eng.FistaOptions(lipschitz=2.9908e5, max_iterations=k, gap_tolerance=1e-300, stop_on_gap=False)
eng.solve_relaxation(inst, opts=o(W), return_device=True)
torch.cuda.synchronize()
for i in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = eng.solve_relaxation(inst, opts=o(K), return_device=True)
    e1.record()
    torch.cuda.synchronize()
    print(f"solve {i}: {e0.elapsed_time(e1):.3f} ms for {r.iterations} its -> {r.iterations / e0.elapsed_time(e1) * 1e3:.0f} it/s",
          flush=True)
