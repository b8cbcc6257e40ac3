"""Benchmark of the B200 dual-bound engine (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one restarted-FISTA iteration of the perspective relaxation on the
workload BASELINE.json's metric is quoted on (configs[1] = C2: least squares,
fp64, n = p = 16000, Toeplitz rho 0.7, k=20, M=2, lambda2=0.1; synthetic data
from the reference's generator with the paper's protocol).  X is 2.05 GB,
larger than the 126 MB L2, so every pass streams HBM.

ours       value  = K iterations / device time of a K-iteration solve with X resident
                    (stop_on_gap=False so exactly K iterations run, bound checks included)
           e2e    = iterations / time of full solves to the C2 target (relative gap
                    <= 1e-6) through solve_relaxation on an instance whose X lives
                    in pinned host memory (H2D of X and y + D2H of beta inside)
reference  the CPU oracle port of the reference solver (oracle/l0_oracle.py, numpy +
           C PAVA, all host threads), K iterations of the same workload
N > 1      node sharding (default): each GPU runs its own branch-and-bound node of C2
           (independent units, no collective, "weak"); --shard rows splits C2's rows
           over the ranks with the engine's NCCL all-reduce each iteration ("strong").
"""

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOAD = "C2"
# injected step constant 2 * 1.01 * lambda_max(X^T X) for C2 (SURVEY.md §8(d):
# Lanczos 2.99073e5), rounded up so it stays a valid Lipschitz bound
L_C2 = 2.9908e5
REL_GAP = 1e-6
TF32_DENSE_PEAK = 1100.0   # TFLOP/s, B200 dense TF32 (B200_PROFILING.md)
METRIC = "FISTA iters/sec (C2 perspective relaxation; N>1: one branch-and-bound node per GPU)"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def make_inputs(scale):
    from paper_2502_09502_b200 import data
    t0 = time.time()
    cd = data.make_config(WORKLOAD, scale=scale)
    log(f"[bench] generated {WORKLOAD} n={cd.n} p={cd.p} in {time.time() - t0:.1f}s")
    return cd


def base_config(cd, n_gpus):
    return {"workload": "C2: least-squares root perspective relaxation, n=p=%d, Toeplitz rho=0.7, "
                        "k=20, M=2, lambda2=0.1, SNR=5" % cd.n,
            "n": cd.n, "p": cd.p, "k": cd.k, "M": cd.M, "lambda2": cd.lambda2,
            "x_bytes": int(cd.X.nbytes), "lipschitz": L_C2,
            "l2_policy": "inputs larger than L2 (X = %.2f GB vs 126 MB)" % (cd.X.nbytes / 1e9),
            "parallelism": "rows%d" % n_gpus if n_gpus > 1 else "single"}


# ---------------------------------------------------------------------------
# clocks (nvidia-smi sampled during the timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic():
    """dram bytes (read + write) per launch of each kernel, from the committed ncu
    --set full captures (profiles/ncu_summary.json)."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return {k: v.get("dram_bytes_per_launch") for k, v in d.get("kernels", {}).items()}
    except Exception:
        return {}


# ---------------------------------------------------------------------------
# CPU baseline (oracle port of the reference solver)
# ---------------------------------------------------------------------------
def cpu_baseline(cd, iters, warm=2):
    import threadpoolctl
    from oracle import l0_oracle
    X = cd.X if cd.X.dtype == np.float64 else cd.X.astype(np.float64)
    cores = os.cpu_count()
    with threadpoolctl.threadpool_limits(cores):
        l0_oracle.fista(X, cd.y, cd.loss, cd.k, cd.M, cd.lambda2, L=L_C2, max_iter=warm,
                        gap_tol=1e-300, stop_on_gap=False)
        t0 = time.perf_counter()
        l0_oracle.fista(X, cd.y, cd.loss, cd.k, cd.M, cd.lambda2, L=L_C2, max_iter=iters,
                        gap_tol=1e-300, stop_on_gap=False)
        dt = time.perf_counter() - t0
    return {"value": iters / dt, "unit": "iters/s", "cores": cores, "kind": "port",
            "sample": f"{iters} FISTA iterations of {WORKLOAD} (after {warm} warm-up) with the "
                      f"numpy/OpenBLAS + C-PAVA oracle port, {cores} threads, {dt:.2f}s"}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    cd = make_inputs(args.scale)
    cb = cpu_baseline(cd, args.steps, warm=args.warmup)
    line = {"metric": METRIC, "value": cb["value"],
            "unit": "iters/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 / cb["value"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference generator, seed 0)",
            "config": base_config(cd, 1), "impl": "reference", "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "iters/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# batched nodes (C4): tensor-core roofline
# ---------------------------------------------------------------------------
def tf32_peak(seconds=1.5):
    """cuBLAS TF32 dense throughput on this GPU (torch.matmul 8192^3, fp32 inputs,
    TF32 math): burst (best) and sustained (back to back) TFLOP/s."""
    import torch
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        n = 8192
        a = torch.randn(n, n, device="cuda")
        b = torch.randn(n, n, device="cuda")
        for _ in range(3):
            a @ b
        torch.cuda.synchronize()
        best = 0.0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(10):
            e0.record(); a @ b; e1.record(); torch.cuda.synchronize()
            best = max(best, 2 * n ** 3 / (e0.elapsed_time(e1) / 1e3) / 1e12)
        t0 = time.perf_counter(); cnt = 0
        e0.record()
        while time.perf_counter() - t0 < seconds:
            a @ b; cnt += 1
            if cnt % 8 == 0:
                torch.cuda.synchronize()
        e1.record(); torch.cuda.synchronize()
        sustained = 2 * n ** 3 * cnt / (e0.elapsed_time(e1) / 1e3) / 1e12
        return best, sustained
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def run_batched(args):
    """C4: 512 node relaxations (n=20000, p=5000 fp32) advanced together; the two
    X passes per iteration are tcgen05 3xTF32 contractions."""
    import torch
    import paper_2502_09502_b200 as eng
    from paper_2502_09502_b200 import data
    t0 = time.time()
    cd = data.make_config("C4", scale=args.c4_scale, nodes=args.c4_nodes)
    inst = eng.ProblemInstance(cd.X, cd.y, eng.LossKind.SQUARED_ERROR, cd.k, cd.M, cd.lambda2,
                               dtype="fp32")
    nodes = [None] + [eng.NodeState(fixed_one=f1, fixed_zero=f0)
                      for f0, f1 in cd.nodes[:args.c4_nodes - 1]]
    L = eng.lipschitz_constant(inst)
    log(f"[bench] C4 generated + L in {time.time() - t0:.1f}s")
    B, n, p, K = len(nodes), cd.n, cd.p, args.c4_steps
    opts = lambda it, prof: eng.FistaOptions(lipschitz=L, max_iterations=it, stop_on_gap=False,
                                             profile=prof)
    eng.solve_relaxation_batched(inst, nodes, opts=opts(3, False))
    eng.solve_relaxation_batched(inst, nodes, opts=opts(3, True))
    torch.cuda.synchronize()
    clocks = ClockSampler(0)
    clocks.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = eng.solve_relaxation_batched(inst, nodes, opts=opts(K, False), return_device=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    assert all(r.iterations == K for r in reps)
    prof = eng.solve_relaxation_batched(inst, nodes, opts=opts(K, True), return_device=True)[0].stats
    it = prof["profiled_iterations"]
    gt, gf, px = prof["gemm_t_ms"] / it, prof["gemm_f_ms"] / it, prof["prox_ms"] / it
    checks = sum(1 for t in range(1, K + 1) if t == 1 or t % 10 == 0) / K
    useful_f = 2.0 * n * p * B
    useful_t = 2.0 * n * p * B * (1.0 + checks)
    burst, sustained = tf32_peak()
    tensor_f = 3 * useful_f / (gf / 1e3) / 1e12
    tensor_t = 3 * useful_t / (gt / 1e3) / 1e12
    cpu = None
    if not args.no_cpu:
        import threadpoolctl
        from oracle import l0_oracle
        X64 = cd.X.astype(np.float64)
        cores = os.cpu_count()
        nd = nodes[1]
        with threadpoolctl.threadpool_limits(cores):
            l0_oracle.fista(X64, cd.y, cd.loss, cd.k, cd.M, cd.lambda2, L=L, max_iter=1,
                            fixed_one=nd.fixed_one, fixed_zero=nd.fixed_zero, stop_on_gap=False)
            t0 = time.perf_counter()
            l0_oracle.fista(X64, cd.y, cd.loss, cd.k, cd.M, cd.lambda2, L=L, max_iter=5,
                            fixed_one=nd.fixed_one, fixed_zero=nd.fixed_zero, stop_on_gap=False)
            dt = time.perf_counter() - t0
        cpu = {"value": 5 / dt, "unit": "node-iters/s", "cores": cores, "kind": "port",
               "sample": f"5 FISTA iterations of one C4 node (oracle port, {cores} threads)"}
    del inst
    torch.cuda.empty_cache()
    return {"workload": f"C4: {B} node relaxations, n={n}, p={p}, fp32 X, SE, k=10, M=2, "
                        f"lambda2=0.5, cold start, {K} iterations each (lockstep)",
            "metric": "node FISTA iterations/s", "value": B * K / (ms / 1e3),
            "ms_per_batched_iteration": ms / K, "clocks": clk,
            "contraction": "tcgen05 kind::tf32, 3xTF32 (hi/lo split), fp32 TMEM accumulation",
            "roofline": {"bound": "tensor", "unit": "TFLOP/s",
                         "kernel": "tc_gemm_kernel (forward X.Beta step)",
                         "achieved": tensor_f, "peak": TF32_DENSE_PEAK,
                         "frac": tensor_f / TF32_DENSE_PEAK,
                         "peak_source": "B200_PROFILING.md dense TF32 (MEASURED_PEAKS.json has no "
                                        "TF32 entry); measured cuBLAS TF32 8192^3 here: burst "
                                        f"{burst:.0f}, sustained {sustained:.0f}",
                         "cublas_tf32_burst": burst, "cublas_tf32_sustained": sustained,
                         "transpose_achieved": tensor_t, "transpose_frac": tensor_t / TF32_DENSE_PEAK,
                         "useful_tflops_forward": useful_f / (gf / 1e3) / 1e12,
                         "flops_per_forward_launch": 3 * useful_f,
                         "note": "tensor FLOPs count the 3 TF32 products of the hi/lo split"},
            "ms_per_iteration_split": {"gemm_transpose": gt, "prox": px, "gemm_forward": gf},
            "cpu_baseline": cpu}


def run_config(name, iters):
    """One more BASELINE config on one GPU (C1: L2-resident fp64; C3: fp32
    logistic): K fixed iterations un-instrumented (iterations/s), then again
    with per-kernel events (the HBM roofline of the dominant pass)."""
    import torch
    import paper_2502_09502_b200 as eng
    from paper_2502_09502_b200 import data
    t0 = time.time()
    cd = data.make_config(name, scale=1.0)
    inst = eng.ProblemInstance(cd.X, cd.y, eng.LossKind(cd.loss), cd.k, cd.M, cd.lambda2, dtype=cd.dtype)
    # L: the reference's power iteration stops at 500 iterations without converging
    # on C3; 300 power iterations on the GPU, x 1.05
    Xd = torch.from_numpy(cd.X).cuda().double()
    v = torch.randn(Xd.shape[1], device="cuda", dtype=torch.float64, generator=torch.Generator("cuda").manual_seed(0))
    for _ in range(300):
        w = Xd.T @ (Xd @ v)
        lam = float(w.norm())
        v = w / lam
    del Xd, v, w
    torch.cuda.empty_cache()
    L = {"squared_error": 2.0, "logistic": 0.25}[cd.loss] * lam * 1.05
    gen_s = time.time() - t0
    o = lambda k, prof: eng.FistaOptions(lipschitz=L, max_iterations=k, gap_tolerance=1e-300,
                                         stop_on_gap=False, profile=prof)
    eng.solve_relaxation(inst, opts=o(5, False), return_device=True)
    eng.solve_relaxation(inst, opts=o(5, True), return_device=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rep = eng.solve_relaxation(inst, opts=o(iters, False), return_device=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    rep_p = eng.solve_relaxation(inst, opts=o(iters, True), return_device=True)
    st = rep_p.stats
    peak, _ = measured_peak()
    s_el = 8 if cd.dtype == "fp64" else 4
    n, p = cd.n, cd.p
    avg = lambda k: st[k + "_ms"] / max(1, st[k + "_count"])
    xb = n * p * s_el
    if st.get("single_pass"):
        kern = {"kf_fused_s": {"launch_ms": avg("k2"), "achieved_gbs": (xb + 8 * (4 * n + p)) / avg("k2") / 1e6},
                "kr_reduce": {"launch_ms": avg("k1")}, "k3_prox_window": {"launch_ms": avg("k3")}}
        kern["kf_fused_s"]["frac"] = kern["kf_fused_s"]["achieved_gbs"] / peak
    else:
        kern = {"k1_forward": {"launch_ms": avg("k1"), "achieved_gbs": (xb + 8 * (p + 2 * n)) / avg("k1") / 1e6},
                "k2_transpose": {"launch_ms": avg("k2"), "achieved_gbs": (xb + 8 * (3 * n + 5 * p)) / avg("k2") / 1e6},
                "k3_prox_window": {"launch_ms": avg("k3")}}
        for k in ("k1_forward", "k2_transpose"):
            kern[k]["frac"] = kern[k]["achieved_gbs"] / peak
    out = {"config": name, "n": n, "p": p, "dtype": cd.dtype, "loss": cd.loss, "k": cd.k, "M": cd.M,
           "lambda2": cd.lambda2, "lipschitz": L, "iterations": iters,
           "value": iters / (ms / 1e3), "unit": "iters/s", "ms_per_iteration": ms / iters,
           "engine_path": "single_pass" if st.get("single_pass") else "two_pass",
           "x_bytes": xb, "l2_resident": xb < 100e6, "kernels": kern, "peak_gbs": peak,
           "primal": rep.primal_value, "dual": rep.dual_bound, "restarts": rep.restarts,
           "setup_s": gen_s}
    del inst
    torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------------------
# ours
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    world, rank, local = dist_env()
    if world > 1 or args.force_dist:
        return run_ours_sharded(args, world, rank, local)
    torch.cuda.set_device(0)
    import paper_2502_09502_b200 as eng
    eng.native.load()
    cd = make_inputs(args.scale)
    inst = eng.ProblemInstance(cd.X, cd.y, eng.LossKind.SQUARED_ERROR, cd.k, cd.M, cd.lambda2)
    t0 = time.time()
    inst.device_problem()
    torch.cuda.synchronize()
    log(f"[bench] upload {time.time() - t0:.2f}s")
    K, W = args.steps, args.warmup

    def fixed(iters, profile):
        return eng.FistaOptions(lipschitz=L_C2, max_iterations=iters, gap_tolerance=1e-300,
                                stop_on_gap=False, profile=profile, engine_path=args.engine)

    # warm-up: W iterations (graph capture, caches)
    eng.solve_relaxation(inst, opts=fixed(W, True), return_device=True)
    torch.cuda.synchronize()
    # timed region: exactly K iterations, CUDA events, clocks sampled
    clocks = ClockSampler(0)
    clocks.start()
    time.sleep(0.3)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    start.record()
    rep = eng.solve_relaxation(inst, opts=fixed(K, False), return_device=True)
    end.record()
    torch.cuda.synchronize()
    ms = start.elapsed_time(end)
    assert rep.iterations == K, rep.iterations
    value = K / (ms / 1e3)
    # the same K iterations again with CUDA events around every kernel inside the
    # graphs (on the engine's stream): the per-launch durations behind the
    # roofline.  The events add ~10 us of graph nodes per iteration, so the
    # headline value above comes from the un-instrumented run.
    start.record()
    rep = eng.solve_relaxation(inst, opts=fixed(K, True), return_device=True)
    end.record()
    torch.cuda.synchronize()
    ms_prof = start.elapsed_time(end)
    clk = clocks.stop()
    assert rep.iterations == K, rep.iterations
    st = rep.stats
    log(f"[bench] {K} its in {ms:.2f} ms -> {value:.1f} it/s; k1 {st['k1_ms'] / max(1, st['k1_count']):.4f} "
        f"ms k2 {st['k2_ms'] / max(1, st['k2_count']):.4f} ms k3 {st['k3_ms'] / max(1, st['k3_count']):.4f} ms")

    # roofline of the dominant kernel (algorithmic bytes / measured launch time)
    peak, peak_src = measured_peak()
    s = 8
    n, p = cd.n, cd.p
    k1_avg = st["k1_ms"] / max(1, st["k1_count"])
    k2_avg = st["k2_ms"] / max(1, st["k2_count"])
    k3_avg = st["k3_ms"] / max(1, st["k3_count"])
    single = bool(st.get("single_pass"))
    traffic = ncu_traffic()
    if single:
        # KF reads X once: both gradient candidates, X^T zeta and u_t from one pass
        kf_bytes = n * p * s + 8 * (4 * n + p)        # X, y, u_{t-1}, u_t (write), beta slice
        dom, dom_bytes, dom_ms = "kf_fused_s", kf_bytes, k2_avg
        others = {"kr_reduce_epilogue": {"launch_ms": k1_avg},
                  "k3_prox_window": {"launch_ms": k3_avg}}
    else:
        k2_bytes = n * p * s + 8 * (3 * n + 5 * p)     # X, u_t, u_t-1, y, beta_t, beta_t-1, gamma, key
        k1_bytes = n * p * s + 8 * (p + 2 * n)          # X, beta, y, u
        dom = "k2_transpose" if st["k2_ms"] >= st["k1_ms"] else "k1_forward"
        dom_bytes, dom_ms = (k2_bytes, k2_avg) if dom == "k2_transpose" else (k1_bytes, k1_avg)
        others = {"k1_forward": {"launch_ms": k1_avg, "achieved_gbs": k1_bytes / (k1_avg / 1e3) / 1e9,
                                 "frac": k1_bytes / (k1_avg / 1e3) / 1e9 / peak},
                  "k2_transpose": {"launch_ms": k2_avg, "achieved_gbs": k2_bytes / (k2_avg / 1e3) / 1e9,
                                   "frac": k2_bytes / (k2_avg / 1e3) / 1e9 / peak},
                  "k3_prox_pava_envelope": {"launch_ms": k3_avg}}
    achieved = dom_bytes / (dom_ms / 1e3) / 1e9
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                "unit": "GB/s", "frac": achieved / peak, "peak_source": peak_src,
                "traffic": traffic.get(dom), "algorithmic_bytes_per_launch": dom_bytes,
                "launch_ms": dom_ms, "launch_ms_source": "CUDA events around each kernel inside the graphs, "
                "second timed run of the same K iterations (instrumented ms/step %.4f)" % (ms_prof / K),
                "engine": "single pass (X read once per iteration)" if single
                else "two pass", "other_kernels": others,
                "iteration_bytes_2pass": 2 * n * p * s,
                "iteration_rate_vs_2pass_roofline": (2 * n * p * s) / (ms / 1e3 / K) / 1e9 / peak,
                "note": "iteration_rate_vs_2pass_roofline > 1 is possible only because the "
                        "single-pass engine reads X once per iteration" if single else ""}
    # end to end through the public API with host-resident X (pinned)
    Xpin = torch.from_numpy(cd.X).pin_memory()
    e2e_iters, e2e_time = 0, 0.0
    h2d = cd.X.nbytes + cd.y.nbytes
    d2h = cd.p * 8
    e2e_reps = []
    for i in range(args.e2e_solves + (1 if args.e2e_solves > 0 else 0)):
        warm = i == 0          # one untimed warm-up call (process-level one-time costs)
        inst_h = eng.ProblemInstance(Xpin, cd.y, eng.LossKind.SQUARED_ERROR, cd.k, cd.M, cd.lambda2)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = eng.solve_relaxation(inst_h, opts=eng.FistaOptions(
            lipschitz=L_C2, gap_tolerance=1e-300, gap_tolerance_rel=REL_GAP, engine_path=args.engine))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if not warm:
            e2e_iters += r.iterations
            e2e_time += dt
        e2e_reps.append({"iterations": r.iterations, "seconds": dt, "rel_gap": r.gap / abs(r.primal_value),
                         "termination": r.termination.value, "warmup": warm})
        inst_h.release_device()
        del inst_h
    e2e = {"value": e2e_iters / e2e_time if e2e_time > 0 else None, "unit": "iters/s",
           "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h,
           "step": "one solve_relaxation call to relative gap 1e-6 from host (pinned) X",
           "solves": e2e_reps}
    log(f"[bench] e2e {e2e['value']} it/s {e2e_reps}")

    cb = cpu_baseline(cd, args.cpu_iters) if not args.no_cpu else None
    del inst
    torch.cuda.empty_cache()
    batched = None
    if args.c4_nodes > 0:
        try:
            batched = run_batched(args)
            log(f"[bench] C4 {batched['value']:.0f} node-it/s {batched['ms_per_iteration_split']}")
        except Exception as exc:   # reported, never silently dropped
            batched = {"error": repr(exc)}
    others = []
    for name in [c for c in args.configs.split(",") if c and c != "none"]:
        try:
            others.append(run_config(name, args.config_steps))
            log(f"[bench] {name} {others[-1]['value']:.1f} it/s {others[-1]['kernels']}")
        except Exception as exc:   # reported, never silently dropped
            others.append({"config": name, "error": repr(exc)})
    line = {"metric": METRIC,
            "value": value, "unit": "iters/s", "n_gpus": 1, "steps": K, "warmup": W,
            "ms_per_step": ms / K, "higher_is_better": True,
            "scaling": "strong" if args.shard == "rows" else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference generator, seed 0)",
            "config": base_config(cd, 1), "roofline": roofline, "cpu_baseline": cb, "e2e": e2e,
            "gpu_launches": int(st["gpu_launches"]), "clocks": clk,
            "engine_path": "single_pass" if single else "two_pass",
            "restarts": rep.restarts, "final_gap": rep.gap,
            "prox_full_passes": st.get("prox_full_passes"), "topk_fallbacks": st.get("topk_fallbacks"),
            "batched_nodes": batched, "other_configs": others}
    print(json.dumps(line), flush=True)


def run_ours_sharded(args, world, rank, local):
    """N > 1.  Default (--shard nodes): node sharding, the path's independent
    units: every rank holds C2's X and runs K iterations of
    its own branch-and-bound node (rank 0 the root, the others seeded
    fixed-zero/fixed-one sets), no data-path collective; value = node
    iterations of all ranks / max-over-ranks device time ("weak").
    --shard rows: C2's rows split over the ranks with the engine's NCCL
    all-reduce of the gradient each iteration ("strong")."""
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2502_09502_b200 import distributed as shard
    import paper_2502_09502_b200 as eng
    from paper_2502_09502_b200 import data
    eng.native.load()
    cd = make_inputs(args.scale)
    K, W = args.steps, args.warmup
    opts = lambda it: eng.FistaOptions(lipschitz=L_C2, max_iterations=it, gap_tolerance=1e-300,
                                       stop_on_gap=False, engine_path=args.engine)
    if args.shard == "rows":
        r0, r1 = shard.row_range(cd.n, world, rank)
        inst = shard.ShardedProblem(cd.X[r0:r1], cd.y[r0:r1], eng.LossKind.SQUARED_ERROR, cd.k,
                                    cd.M, cd.lambda2, n_global=cd.n)
        solve = lambda it: shard.solve_relaxation_sharded(inst, opts=opts(it))
        scaling, units_per_step, par = "strong", 1, "rows%d" % world
    else:
        inst = eng.ProblemInstance(cd.X, cd.y, eng.LossKind.SQUARED_ERROR, cd.k, cd.M, cd.lambda2)
        sets = data.random_nodes(cd.p, world, seed=1)
        node = None if rank == 0 else eng.NodeState(fixed_one=sets[rank][1], fixed_zero=sets[rank][0])
        solve = lambda it: eng.solve_relaxation(inst, node, opts=opts(it), return_device=True)
        scaling, units_per_step, par = "weak", world, "nodes%d" % world
    solve(W)
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    rep = solve(K)
    end.record()
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    ms = torch.tensor([start.elapsed_time(end)], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    launches = torch.tensor([float(rep.stats["gpu_launches"])], device="cuda")
    dist.all_reduce(launches)
    if rank == 0:
        cfg = base_config(cd, world)
        cfg["parallelism"] = par
        line = {"metric": METRIC,
                "value": units_per_step * K / (ms / 1e3), "unit": "iters/s", "n_gpus": world,
                "steps": K, "warmup": W, "ms_per_step": ms / K, "higher_is_better": True,
                "scaling": scaling, "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (reference generator, seed 0)", "config": cfg,
                "gpu_launches": int(launches.item()),
                "engine_path": "single_pass" if rep.stats.get("single_pass") else "two_pass"}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scale", type=float, default=1.0, help="shrink C2 (testing only)")
    ap.add_argument("--e2e-solves", type=int, default=2)
    ap.add_argument("--cpu-iters", type=int, default=10)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--engine", default="auto", choices=["auto", "two_pass", "single_pass"])
    ap.add_argument("--force-dist", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--shard", default="nodes", choices=["nodes", "rows"],
                    help="N > 1: independent node relaxations per GPU (weak) or C2's rows (strong)")
    ap.add_argument("--c4-nodes", type=int, default=512, help="batched-node section (0: skip)")
    ap.add_argument("--c4-steps", type=int, default=100)
    ap.add_argument("--c4-scale", type=float, default=1.0)
    ap.add_argument("--configs", default="C1,C3", help="extra single-GPU configs reported under other_configs")
    ap.add_argument("--config-steps", type=int, default=200)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
