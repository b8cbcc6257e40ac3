"""Phase timing of the prox kernel (build with L0_PROBE=1)."""
import ctypes, sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2502_09502_b200 as eng
from paper_2502_09502_b200 import data
eng.native.load()
cd = data.make_config("C2", scale=float(sys.argv[1]) if len(sys.argv) > 1 else 1.0)
inst = eng.ProblemInstance(cd.X, cd.y, eng.LossKind.SQUARED_ERROR, cd.k, cd.M, cd.lambda2)
for its in (5, 23, 40):
    rep = eng.solve_relaxation(inst, opts=eng.FistaOptions(lipschitz=2.9908e5, max_iterations=its,
                               gap_tolerance=1e-300, stop_on_gap=False, chunk_iterations=1))
    buf = (ctypes.c_int64 * 16)()
    eng.native.lib().l0_debug_probe(inst.device_problem().handle, buf)
    v = list(buf)
    names = ["start", "dual", "gather+offs", "merge", "append", "search", "->scatter", "scatter", "g+theta"]
    d = [(names[i], (v[i] - v[i - 1]) / 1.965e3) for i in range(1, 9) if v[i] and v[i - 1]]
    print(its, rep.stats, [(n, round(x, 2)) for n, x in d], "total us", (v[8] - v[0]) / 1.965e3)
