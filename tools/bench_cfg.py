"""Iterations/s of a BASELINE config on both engine paths:
python tools/bench_cfg.py C3 [scale] [iters]"""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2502_09502_b200 as eng
from paper_2502_09502_b200 import data

name = sys.argv[1]
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 100
t0 = time.time()
cd = data.make_config(name, scale=scale)
inst = eng.ProblemInstance(cd.X, cd.y, eng.LossKind(cd.loss), cd.k, cd.M, cd.lambda2, dtype=cd.dtype)
Xd = torch.from_numpy(cd.X).cuda()
Xd = Xd.double() if Xd.numel() < 2e9 else Xd          # fp32 power iteration for huge X
v = torch.randn(Xd.shape[1], device="cuda", dtype=Xd.dtype)
for _ in range(300):                    # power iteration (the reference's 500-it cap fails here)
    w = Xd.T @ (Xd @ v)
    lam = float(w.norm())
    v = w / lam
del Xd
torch.cuda.empty_cache()
L = {"squared_error": 2.0, "logistic": 0.25}[cd.loss] * lam * 1.05
print(f"{name} n={cd.n} p={cd.p} {cd.dtype} {cd.loss} gen+L {time.time()-t0:.1f}s L={L:.6g}", flush=True)
res = {}
paths = sys.argv[4].split(",") if len(sys.argv) > 4 else ["two_pass", "single_pass"]
for path in paths:
    o = lambda k: eng.FistaOptions(lipschitz=L, max_iterations=k, stop_on_gap=False, gap_tolerance=1e-300,
                                   engine_path=path, profile=True)
    try:
        eng.solve_relaxation(inst, opts=o(3), return_device=True)
    except Exception as exc:
        print(path, "unavailable:", exc)
        continue
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = eng.solve_relaxation(inst, opts=o(iters), return_device=True)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    st = r.stats
    res[path] = r
    print(f"{path}: {iters/(ms/1e3):.1f} it/s ({ms/iters:.3f} ms/it) k1 {st['k1_ms']/max(1,st['k1_count']):.4f} "
          f"k2 {st['k2_ms']/max(1,st['k2_count']):.4f} k3 {st['k3_ms']/max(1,st['k3_count']):.4f} "
          f"obj {r.primal_value:.12g} dual {r.dual_bound:.12g} cs {st["cluster_size"]} full_prox {st["prox_full_passes"]} topk_fb {st["topk_fallbacks"]} restarts {r.restarts}", flush=True)
if len(res) == 2:
    a, b = res["two_pass"], res["single_pass"]
    print("rel obj diff", abs(a.primal_value - b.primal_value) / abs(a.primal_value),
          "beta diff", float((a.beta - b.beta).abs().max()))
