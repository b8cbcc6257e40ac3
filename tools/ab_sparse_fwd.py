"""A/B of the batched engine's forward contraction on C4: support-compacted
(default) vs dense (L0_SPARSE_FWD=0).  Runs both in subprocesses, prints the
per-iteration time and the largest relative objective / bound difference.

    python tools/ab_sparse_fwd.py [scale] [nodes] [iters]
"""
import json, os, subprocess, sys

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, ".")
    import time
    import numpy as np
    import torch
    import paper_2502_09502_b200 as eng
    from paper_2502_09502_b200.data import make_config
    scale, count, iters, out = float(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
    cfg = make_config("C4", scale=scale, nodes=count)
    inst = eng.ProblemInstance(cfg.X, cfg.y, eng.LossKind.SQUARED_ERROR, cfg.k, cfg.M, cfg.lambda2, dtype="fp32")
    nodes = [None] + [eng.NodeState(fixed_one=f1, fixed_zero=f0) for f0, f1 in cfg.nodes[:count - 1]]
    L = eng.lipschitz_constant(inst, method="lanczos")
    o = lambda it, prof=False: eng.FistaOptions(max_iterations=it, stop_on_gap=False, lipschitz=L, profile=prof)
    eng.solve_relaxation_batched(inst, nodes, opts=o(3))
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        reps = eng.solve_relaxation_batched(inst, nodes, opts=o(iters))
        ts.append(time.perf_counter() - t0)
    prof = eng.solve_relaxation_batched(inst, nodes, opts=o(iters, True))[0].stats
    dt = min(ts)
    np.savez(out, primal=[r.primal_value for r in reps], dual=[r.dual_bound for r in reps],
             beta=np.stack([r.beta for r in reps]))
    it = prof["profiled_iterations"]
    print(json.dumps({"ms_per_it": dt / iters * 1e3, "node_it_s": count * iters / dt,
                      "gemm_t": prof["gemm_t_ms"] / it, "prox": prof["prox_ms"] / it,
                      "gemm_f": prof["gemm_f_ms"] / it}), flush=True)
    sys.exit(0)

import numpy as np
scale = sys.argv[1] if len(sys.argv) > 1 else "1.0"
count = sys.argv[2] if len(sys.argv) > 2 else "512"
iters = sys.argv[3] if len(sys.argv) > 3 else "100"
os.makedirs("gpurun_out", exist_ok=True)
res = {}
for mode in ("1", "0"):
    env = dict(os.environ, L0_SPARSE_FWD=mode)
    out = f"gpurun_out/ab_sparse_{mode}.npz"
    r = subprocess.run([sys.executable, __file__, "--child", scale, count, iters, out], env=env,
                       capture_output=True, text=True)
    print(f"L0_SPARSE_FWD={mode}: rc={r.returncode} {r.stdout.strip()} {r.stderr[-2000:] if r.returncode else ''}")
    res[mode] = np.load(out) if r.returncode == 0 else None
if res["1"] is not None and res["0"] is not None:
    a, b = res["1"], res["0"]
    rel = lambda x, y: float(np.max(np.abs(x - y) / np.maximum(1.0, np.abs(y))))
    print("max rel diff primal", rel(a["primal"], b["primal"]), "dual", rel(a["dual"], b["dual"]),
          "beta", float(np.max(np.abs(a["beta"] - b["beta"]))))
