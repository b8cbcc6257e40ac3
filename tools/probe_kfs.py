"""Per-tile timeline of kf_fused_s (build with L0_PROBE=1): python tools/probe_kfs.py
stamps per tile: 0 fwd start, 1 fwd data ready, 2 fwd partials sent, 3 transpose
partials ready (step's first tile), 4 transpose done."""
import ctypes, sys
sys.path.insert(0, ".")
import numpy as np
import paper_2502_09502_b200 as eng
from paper_2502_09502_b200 import data

cd = data.make_config("C2", scale=1.0)
inst = eng.ProblemInstance(cd.X, cd.y, eng.LossKind.SQUARED_ERROR, cd.k, cd.M, cd.lambda2)
opts = eng.FistaOptions(lipschitz=2.9908e5, max_iterations=3, stop_on_gap=False, gap_tolerance=1e-300,
                        engine_path="single_pass", chunk_iterations=1)
eng.solve_relaxation(inst, opts=opts)
buf = np.zeros(12000)
eng.native.check(eng.native.lib().l0_debug_scratch(inst.device_problem().handle,
                                                   buf.ctypes.data_as(ctypes.c_void_p), 12000))
for c in range(2):
    t = buf[c * 6000:(c + 1) * 6000].reshape(1000, 6)
    t = t[t[:, 0] > 0]
    if len(t) == 0:
        continue
    t = (t - t[0, 0]) / 1e3
    med = lambda v: float(np.median(v))
    print(f"cta{c}: tiles={len(t)} data wait {med(t[:,1]-t[:,0]):.2f} fwd {med(t[:,2]-t[:,1]):.2f} "
          f"period {med(np.diff(t[:,0])):.2f} us")
    st = t[::int(__import__("os").environ.get("TB", "2"))]
    st = st[st[:, 3] > 0]
    print(f"   sent->tr ready {med(st[:,3]-st[:,2]):.2f} tr {med(st[:,4]-st[:,3]):.2f} "
          f"tr period {med(np.diff(st[:,3])):.2f} us")
    for k in list(range(0, 12)) + [100, 101, 102, 103]:
        if k < len(t):
            print("  tile", k, np.round(t[k], 2))
