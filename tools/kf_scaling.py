"""KF launch time vs rows (fixed p): the intercept is the per-launch ramp + drain."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2502_09502_b200 as eng
p = 16000
for n in (4000, 8000, 16000, 32000):
    g = torch.Generator("cuda").manual_seed(n)
    X = torch.randn(n, p, device="cuda", dtype=torch.float64, generator=g)
    y = torch.randn(n, device="cuda", dtype=torch.float64, generator=g).cpu().numpy()
    inst = eng.ProblemInstance(X, y, eng.LossKind.SQUARED_ERROR, 20, 2.0, 0.1)
    L = 2.0 * 1.01 * (n ** 0.5 + p ** 0.5) ** 2
    o = lambda k, prof: eng.FistaOptions(lipschitz=L, max_iterations=k, gap_tolerance=1e-300,
                                         stop_on_gap=False, profile=prof)
    eng.solve_relaxation(inst, opts=o(5, True), return_device=True)
    r = eng.solve_relaxation(inst, opts=o(100, True), return_device=True)
    st = r.stats
    kf = st["k2_ms"] / st["k2_count"]
    print(f"n={n}: KF {kf * 1e3:.1f} us  ({n * p * 8 / kf / 1e6:.0f} GB/s)  single={st['single_pass']}", flush=True)
    del inst, X
    torch.cuda.empty_cache()
