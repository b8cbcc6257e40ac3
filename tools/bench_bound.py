"""Batched fp64 safe lower bound vs the per-node loop on C4's X:
python tools/bench_bound.py [nodes] [scale]"""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2502_09502_b200 as eng
from paper_2502_09502_b200 import data

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 64
cd = data.make_config("C4", scale=float(sys.argv[2]) if len(sys.argv) > 2 else 1.0)
inst = eng.ProblemInstance(cd.X, cd.y, eng.LossKind(cd.loss), cd.k, cd.M, cd.lambda2, dtype=cd.dtype)
rng = np.random.default_rng(0)
nodes = [eng.NodeState(fixed_one=tuple(int(v) for v in rng.choice(cd.p, 2, replace=False)[:1]),
                       fixed_zero=()) for _ in range(nb)]
betas = rng.standard_normal((nb, cd.p)) * 0.1
bd = torch.from_numpy(betas).cuda()
eng.safe_lower_bound_batched(inst, bd, nodes)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    got = eng.safe_lower_bound_batched(inst, bd, nodes)
tb = (time.perf_counter() - t0) / 5
t0 = time.perf_counter()
single = [eng.safe_lower_bound(inst, bd[j], nodes[j]) for j in range(nb)]
ts = time.perf_counter() - t0
err = max(abs(a - b) / max(1.0, abs(b)) for a, b in zip(got, single))
flops = 2 * 2.0 * cd.n * cd.p * nb
print(f"C4 n={cd.n} p={cd.p} {cd.dtype} nodes={nb}: batched {tb*1e3:.2f} ms ({flops/tb/1e12:.1f} TF/s fp64), "
      f"per-node loop {ts*1e3:.2f} ms, speed-up {ts/tb:.1f}x, max rel diff {err:.2e}")
