"""Per-tile timeline of kf_fused_s (build with L0_PROBE=1):
python tools/probe_kfs.py [config] [scale]
stamps per tile (CTA 0 and CTA cs-1): 0 fwd start, 1 tile landed, 2 partials
sent, 3 gather start (partials complete), 4 accumulated, 5 refill issued (of
tile k + S, stamped at k)."""
import ctypes, os, sys
sys.path.insert(0, ".")
import numpy as np
import paper_2502_09502_b200 as eng
from paper_2502_09502_b200 import data

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
L = {"C1": 10.0689, "C2": 2.9908e5, "C3": 60296.1, "C4": 1.0e5, "C5": 6.5587e6}[name]
cd = data.make_config(name, scale=scale)
inst = eng.ProblemInstance(cd.X, cd.y, eng.LossKind(cd.loss), cd.k, cd.M, cd.lambda2, dtype=cd.dtype)
opts = eng.FistaOptions(lipschitz=L, max_iterations=3, stop_on_gap=False, gap_tolerance=1e-300,
                        engine_path="single_pass", chunk_iterations=1)
rep = eng.solve_relaxation(inst, opts=opts)
print(name, scale, "cluster", rep.stats["cluster_size"])
buf = np.zeros(12000)
eng.native.check(eng.native.lib().l0_debug_scratch(inst.device_problem().handle,
                                                   buf.ctypes.data_as(ctypes.c_void_p), 12000))
med = lambda v: float(np.nanmedian(v)) if len(v) else float("nan")
for c in range(2):
    t = buf[c * 6000:(c + 1) * 6000].reshape(1000, 6)
    nt = int(np.sum(t[:, 0] > 0))
    if nt == 0:
        continue
    t = t[:nt]
    t = np.where(t > 0, (t - t[0, 0]) / 1e3, np.nan)
    lo, hi = min(20, nt // 4), max(nt - 20, nt // 2)
    s = t[lo:hi]
    print(f"cta{c}: tiles={nt} steady [{lo},{hi}) period fwd {med(np.diff(s[:,0])):.3f} "
          f"gather {med(np.diff(s[:,3])):.3f} acc {med(np.diff(s[:,4])):.3f} us")
    print(f"   wait landed {med(s[:,1]-s[:,0]):.3f} fwd compute {med(s[:,2]-s[:,1]):.3f} "
          f"sent->gather {med(s[:,3]-s[:,2]):.3f} gather->acc done {med(s[:,4]-s[:,3]):.3f} us")
    S = None
    for k in range(1, 20):   # ring depth: refill stamp of tile k issued for tile k+S
        pass
    life = []
    for k in range(lo, hi):
        # tile k landed at t[k,1]; its stage was refilled at t[k-S,5] -- report landed - accumulated(k-1)
        life.append(t[k, 4] - t[k, 1])
    print(f"   landed->accumulated {med(life):.3f} us; refill->landed (k vs stamp5 of k-S unknown S)")
    for k in list(range(0, 6)) + [lo, lo + 1, lo + 2, lo + 3]:
        if k < nt:
            print("  tile", k, np.round(t[k], 3))
