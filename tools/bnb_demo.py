"""Branch-and-bound certification demo on a synthetic instance:
python tools/bnb_demo.py [n] [p] [k] [snr]"""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2502_09502_b200 as eng
from paper_2502_09502_b200 import data
from paper_2502_09502_b200.bnb import BnBOptions, certify

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
p = int(sys.argv[2]) if len(sys.argv) > 2 else 500
k = int(sys.argv[3]) if len(sys.argv) > 3 else 5
snr = float(sys.argv[4]) if len(sys.argv) > 4 else 5.0
X, y, bt = data.synthetic(n, p, k, sigma=0.5, snr=snr, seed=0)
inst = eng.ProblemInstance(X, y, eng.LossKind.SQUARED_ERROR, k, 2.0, 1.0)
t0 = time.time()
L = 2.0 * 1.01 * float(np.linalg.norm(X, 2) ** 2)
opts = BnBOptions(gap_tolerance=1e-4, batch_size=64,
                  relaxation=eng.FistaOptions(max_iterations=3000, lipschitz=L, gap_tolerance=1e-6))
certify(inst, BnBOptions(node_limit=1, relaxation=opts.relaxation))   # warm-up (engine setup)
t0 = time.time()
cert = certify(inst, opts)
dt = time.time() - t0
print(f"n={n} p={p} k={k} snr={snr}: status={cert.status.value} nodes={cert.nodes_explored} "
      f"incumbent={cert.incumbent_objective:.6f} lower={cert.global_lower_bound:.6f} "
      f"gap={cert.gap_relative:.2e} time={dt:.2f}s support={np.flatnonzero(cert.incumbent_beta).tolist()} "
      f"true={np.flatnonzero(bt).tolist()}")
