"""One C2 solve of K iterations after warm-up (for ncu launch lists):
python tools/one_solve.py [K] [scale]"""
import sys
sys.path.insert(0, ".")
import torch
import paper_2502_09502_b200 as eng
from paper_2502_09502_b200 import data

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
cd = data.make_config("C2", scale=float(sys.argv[2]) if len(sys.argv) > 2 else 1.0)
inst = eng.ProblemInstance(cd.X, cd.y, eng.LossKind.SQUARED_ERROR, cd.k, cd.M, cd.lambda2)
o = lambda k: eng.FistaOptions(lipschitz=2.9908e5, max_iterations=k, gap_tolerance=1e-300, stop_on_gap=False)
eng.solve_relaxation(inst, opts=o(K), return_device=True)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
rep = eng.solve_relaxation(inst, opts=o(K), return_device=True)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print(K, rep.iterations, rep.stats["gpu_launches"])
