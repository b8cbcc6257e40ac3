"""One single-pass solve of a BASELINE config, one iteration per graph replay,
for ncu captures of a mid-solve KF launch:
ncu -k regex:kf_fused_s -s 10 -c 1 python tools/ncu_cfg_kf.py C3 [scale]"""
import sys
sys.path.insert(0, ".")
import torch
import paper_2502_09502_b200 as eng
from paper_2502_09502_b200 import data

cd = data.make_config(sys.argv[1], scale=float(sys.argv[2]) if len(sys.argv) > 2 else 1.0)
inst = eng.ProblemInstance(cd.X, cd.y, eng.LossKind(cd.loss), cd.k, cd.M, cd.lambda2, dtype=cd.dtype)
L = {"C1": 10.0689, "C2": 2.9908e5, "C3": 60296.1, "C4": 1.0e5, "C5": 6.5587e6}[sys.argv[1]]
rep = eng.solve_relaxation(inst, opts=eng.FistaOptions(lipschitz=L, max_iterations=30, stop_on_gap=False,
                                                       gap_tolerance=1e-300, chunk_iterations=1))
torch.cuda.synchronize()
print(sys.argv[1], rep.iterations, rep.primal_value, rep.stats)
