"""Per-tile timeline of the single-pass kernel (build with L0_PROBE=1):
python tools/probe_kf.py  -> forward / transpose durations and lags."""
import ctypes, os, sys
sys.path.insert(0, ".")
import numpy as np
import torch
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
    valid = t[:, 0] > 0
    t = t[valid]
    if len(t) == 0:
        continue
    t0 = t[0, 0]
    t = (t - t0) / 1e3  # us
    fwd = t[:, 1] - t[:, 0]
    tr = t[:, 3] - t[:, 2]
    lag = t[:, 2] - t[:, 1]
    gap_f = np.diff(t[:, 0])
    gap_t = np.diff(t[:, 2])
    wait_full = t[:, 4] - t[:, 0]
    dots = t[:, 5] - t[:, 4]
    send = t[:, 1] - t[:, 5]
    print(f"  fwd phases med: wait data {np.median(wait_full):.2f} dots+reduce {np.median(dots):.2f} send {np.median(send):.2f} us")
    print(f"cta{c}: tiles={len(t)} span={t[-1,3]:.1f}us fwd dur med {np.median(fwd):.2f} "
          f"fwd period med {np.median(gap_f):.2f} tr dur med {np.median(tr):.2f} tr period med "
          f"{np.median(gap_t):.2f} lag(fwd end->tr start) med {np.median(lag):.2f} us")
    for k in list(range(0, 6)) + [100, 101, 102]:
        if k < len(t):
            print("  tile", k, np.round(t[k], 2))
