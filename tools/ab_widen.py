"""A/B of the fp32 KF widening modes (L0_FZ_WIDEN: 0 = F2F everywhere, 1 =
integer rebias in the forward warps, 2 = in the accumulate warps, 3 = both):
python tools/ab_widen.py C3 [scale] [iters] [modes]
Results must be bitwise identical across modes (the rebias is exact)."""
import os, sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2502_09502_b200 as eng
from paper_2502_09502_b200 import data

name = sys.argv[1]
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 100
modes = [int(m) for m in (sys.argv[4] if len(sys.argv) > 4 else "0,1,2,3").split(",")]
cd = data.make_config(name, scale=scale)
L = {"C3": 60296.1, "C5": 6.5587e6, "C2": 2.9908e5}[name]
ref = None
for m in modes:
    os.environ["L0_FZ_WIDEN"] = str(m)
    inst = eng.ProblemInstance(cd.X, cd.y, eng.LossKind(cd.loss), cd.k, cd.M, cd.lambda2, dtype=cd.dtype)
    f32 = os.environ.get("FP32_FORWARD") == "1"
    o = lambda k: eng.FistaOptions(lipschitz=L, max_iterations=k, stop_on_gap=False, gap_tolerance=1e-300,
                                   engine_path="single_pass", profile=os.environ.get("PROFILE", "1") == "1",
                                   fp32_forward=f32)
    eng.solve_relaxation(inst, opts=o(3))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = eng.solve_relaxation(inst, opts=o(iters))
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    st = r.stats
    kf = st.get('k2_ms', 0.0) / max(1, st.get('k2_count', 0)) or 1e-9
    xb = cd.n * cd.p * cd.X.itemsize
    same = "" if ref is None else (f" bitwise={np.array_equal(ref.beta, r.beta) and ref.primal_value == r.primal_value and ref.dual_bound == r.dual_bound}")
    print(f"{name} widen={m}: {iters/(ms/1e3):.1f} it/s ({ms/iters:.3f} ms/it) kf {kf:.4f} ms "
          f"({xb/kf/1e6:.0f} GB/s) k3 {st.get('k3_ms', 0.0)/max(1,st.get('k3_count', 0)):.4f} obj {r.primal_value:.15g}{same}",
          flush=True)
    ref = ref or r
    del inst
    torch.cuda.empty_cache()
