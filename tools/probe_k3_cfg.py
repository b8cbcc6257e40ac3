"""K3 phase timing for any config (build with L0_PROBE=1):
python tools/probe_k3_cfg.py C3 [scale]"""
import ctypes, os, sys
sys.path.insert(0, ".")
import torch
import paper_2502_09502_b200 as eng
from paper_2502_09502_b200 import data
eng.native.load()
name = sys.argv[1]
cd = data.make_config(name, scale=float(sys.argv[2]) if len(sys.argv) > 2 else 1.0)
inst = eng.ProblemInstance(cd.X, cd.y, eng.LossKind(cd.loss), cd.k, cd.M, cd.lambda2, dtype=cd.dtype)
Xd = torch.from_numpy(cd.X).cuda().double()
v = torch.randn(Xd.shape[1], device="cuda", dtype=torch.float64)
for _ in range(200):
    w = Xd.T @ (Xd @ v); lam = float(w.norm()); v = w / lam
del Xd
L = {"squared_error": 2.0, "logistic": 0.25}[cd.loss] * lam * 1.05
names = ["start", "dual", "gather+offs", "merge", "append", "search", "->scatter", "scatter", "g+theta"]
for its in (2, 5, 11, 23, 40, 80):
    rep = eng.solve_relaxation(inst, opts=eng.FistaOptions(lipschitz=L, max_iterations=its, engine_path=os.environ.get("ENGINE", "two_pass"),
                               gap_tolerance=1e-300, stop_on_gap=False, chunk_iterations=1))
    buf = (ctypes.c_int64 * 16)()
    eng.native.lib().l0_debug_probe(inst.device_problem().handle, buf)
    v = list(buf)
    d = [(names[i], (v[i] - v[i - 1]) / 1.965e3) for i in range(1, 9) if v[i] and v[i - 1]]
    extra = ""
    print(its, extra, {k: rep.stats[k] for k in ("prox_full_passes", "topk_fallbacks")},
          [(n, round(x, 2)) for n, x in d], "total us", round((v[8] - v[0]) / 1.965e3, 1), flush=True)
