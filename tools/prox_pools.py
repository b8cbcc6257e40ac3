"""Per-iteration PAVA pool [a*, c*], sorted-prefix length and K3 path over the
first iterations of a BASELINE config (the engine's prox record ring):
python tools/prox_pools.py [C2|C3|C5] [scale] [iters]"""
import sys
sys.path.insert(0, ".")
import torch
import paper_2502_09502_b200 as eng
from paper_2502_09502_b200 import data

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 12
eng.native.load()
cd = data.make_config(name, scale=scale)
inst = eng.ProblemInstance(cd.X, cd.y, eng.LossKind(cd.loss), cd.k, cd.M, cd.lambda2, dtype=cd.dtype)
L = {"C2": 2.9908e5, "C3": 60296.1, "C5": 6.5587e6}[name]
dp = inst.device_problem()
HEAD, W = 8, 8
ring = torch.full((iters + 2, HEAD + W), -2, dtype=torch.int32, device=dp.X.device)
lib = eng.native.lib()
eng.native.check(lib.l0_problem_set_prox_record(dp.handle, ring.data_ptr(), iters + 2, W))
rep = eng.solve_relaxation(inst, opts=eng.FistaOptions(lipschitz=L, max_iterations=iters, gap_tolerance=1e-300,
                                                       stop_on_gap=False))
eng.native.check(lib.l0_problem_set_prox_record(dp.handle, None, 0, 0))
torch.cuda.synchronize()
r = ring.cpu().numpy()
for row in sorted(r.tolist(), key=lambda x: x[0]):
    if row[0] < 0:
        continue
    print(f"iter {row[0]:3d} how {row[1]} pool {row[2]} a* {row[3]:6d} c* {row[4]:6d} len {row[5]:6d} "
          f"path {row[6]} nfree {row[7]}")
