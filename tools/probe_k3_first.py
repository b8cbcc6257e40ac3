"""Phase timing of the prox kernel on the first iterations of a C2 solve
(build with L0_PROBE=1): each solve of K iterations leaves the stamps of
iteration K's prox launch (the final bound-only launch rewrites stamp 0 only).
python tools/probe_k3_first.py [C2|C3|C5] [scale]"""
import sys
sys.path.insert(0, ".")
import paper_2502_09502_b200 as eng
from paper_2502_09502_b200 import data
import ctypes
eng.native.load()
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cd = data.make_config(name, scale=float(sys.argv[2]) if len(sys.argv) > 2 else 1.0)
inst = eng.ProblemInstance(cd.X, cd.y, eng.LossKind(cd.loss), cd.k, cd.M, cd.lambda2, dtype=cd.dtype)
L = {"C2": 2.9908e5, "C3": 60296.1, "C5": 6.5587e6}[name]
names = ["start", "dual", "gather+offs", "merge", "append", "search", "->scatter", "scatter", "g+theta"]
for its in (1, 2, 3, 4, 5, 8, 30):
    rep = eng.solve_relaxation(inst, opts=eng.FistaOptions(lipschitz=L, max_iterations=its, engine_path="single_pass",
                               gap_tolerance=1e-300, stop_on_gap=False, chunk_iterations=1))
    buf = (ctypes.c_int64 * 16)()
    eng.native.lib().l0_debug_probe(inst.device_problem().handle, buf)
    v = list(buf)
    d = [(names[i], round((v[i] - v[i - 1]) / 1.965e3, 1)) for i in range(2, 9) if v[i] and v[i - 1]]
    print(its, "win_ext", rep.stats.get("win_ext"), "slow", rep.stats.get("prox_full_passes"), d,
          "1->8 us", round((v[8] - v[1]) / 1.965e3, 1), flush=True)
