"""cProfile of a branch-and-bound certification (tools/bnb_demo.py's
instance): where the host time goes.  python tools/bnb_profile.py [n] [p] [k] [snr]"""
import cProfile, pstats, sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2502_09502_b200 as eng
from paper_2502_09502_b200 import data
from paper_2502_09502_b200.bnb import BnBOptions, certify

n = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
p = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
k = int(sys.argv[3]) if len(sys.argv) > 3 else 8
snr = float(sys.argv[4]) if len(sys.argv) > 4 else 3.0
X, y, bt = data.synthetic(n, p, k, sigma=0.5, snr=snr, seed=0)
inst = eng.ProblemInstance(X, y, eng.LossKind.SQUARED_ERROR, k, 2.0, 1.0)
L = 2.0 * 1.01 * float(np.linalg.norm(X, 2) ** 2)
opts = BnBOptions(gap_tolerance=1e-4, batch_size=64,
                  relaxation=eng.FistaOptions(max_iterations=3000, lipschitz=L, gap_tolerance=1e-6))
certify(inst, BnBOptions(node_limit=1, relaxation=opts.relaxation))
t0 = time.time()
pr = cProfile.Profile()
pr.enable()
cert = certify(inst, opts)
pr.disable()
print(f"status={cert.status.value} nodes={cert.nodes_explored} time={time.time() - t0:.2f}s")
pstats.Stats(pr).sort_stats("cumulative").print_stats(22)
