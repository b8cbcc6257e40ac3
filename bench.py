"""Benchmark of the B200 dual-bound engine (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one restarted-FISTA iteration of the perspective relaxation.

N = 1 (headline): configs[1] = C2, least squares, fp64, n = p = 16000,
Toeplitz rho 0.7, k=20, M=2, lambda2=0.1, synthetic data from the reference's
own generator (2.05 GB X, far beyond the 126 MB L2: every pass streams HBM).
    value  = K iterations / device time of a K-iteration solve, X resident
             (stop_on_gap=False so exactly K iterations run, bound checks included)
    e2e    = iterations / time of full solves to the C2 target (relative gap
             <= 1e-6) through solve_relaxation with X in host memory: the
             numpy (pageable) call a drop-in user makes, H2D of X and y and D2H
             of beta inside; the pinned-tensor variant is reported beside it
  sections on the same line: C5 (10^6 x 10^4 fp32, 40 GB, the row-sharding
  config) on one GPU with its own roofline and CPU baseline; C4 batched nodes
  (tcgen05 tensor roofline); C1 and C3.
N > 1 (torchrun, one rank per GPU, NCCL):
    --shard rows (default): C5's rows split over the ranks, each rank
             generating its own rows in HBM; the engine all-reduces the gradient
             over NCCL every iteration ("strong": fixed total work);
    --shard nodes: C4's 512 nodes split over the ranks, each rank one batched
             call on its share (no collective).
reference  the reference's own CPU solver (baseline/_ref, the unmodified
           l0cert.fista.solve_relaxation) on the same config, all host threads;
           the oracle port (oracle/l0_oracle.py) is timed beside it.
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
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/l0_numba_cache")

# injected step constant 2 * 1.01 * lambda_max(X^T X) for C2 (SURVEY.md §8(d):
# Lanczos 2.99073e5), rounded up so it stays a valid Lipschitz bound; the
# package's own Lanczos reproduces it (tests/test_gpu_fullsize.py)
L_C2 = 2.9908e5
REL_GAP = 1e-6
METRIC = "FISTA iters/sec (N=1: C2 perspective relaxation; N>1: C5 rows sharded over the GPUs)"
C2_WORKLOAD = ("C2: least-squares root perspective relaxation, n=p=16000, Toeplitz rho=0.7, "
               "k=20, M=2, lambda2=0.1, SNR=5, fp64")
C5_WORKLOAD = ("C5: least-squares root perspective relaxation, n=1e6, p=1e4 fp32 (40 GB), "
               "Toeplitz rho=0.5, k=25, M=2, lambda2=0.1, SNR=5; rows sharded over the GPUs "
               "with the engine's NCCL all-reduce of the gradient each iteration")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def c2_inputs(scale):
    from paper_2502_09502_b200 import data
    t0 = time.time()
    cd = data.make_config("C2", scale=scale)
    log(f"[bench] generated C2 n={cd.n} p={cd.p} in {time.time() - t0:.1f}s")
    return cd


def c2_config(cd):
    return {"workload": C2_WORKLOAD if cd.n == 16000 else C2_WORKLOAD + f" (scaled to n=p={cd.n})",
            "n": cd.n, "p": cd.p, "k": cd.k, "M": cd.M, "lambda2": cd.lambda2,
            "x_bytes": int(cd.X.nbytes), "lipschitz": L_C2,
            "l2_policy": "inputs larger than L2 (X = %.2f GB vs 126 MB)" % (cd.X.nbytes / 1e9),
            "parallelism": "single"}


def c5_config(n, p, world, shard="rows"):
    return {"workload": C5_WORKLOAD if n == 1_000_000 else C5_WORKLOAD + f" (scaled to n={n})",
            "n": n, "p": p, "k": 25, "M": 2.0, "lambda2": 0.1, "x_bytes": n * p * 4,
            "l2_policy": "inputs larger than L2 (X = %.1f GB vs 126 MB)" % (n * p * 4 / 1e9),
            "parallelism": f"{shard}{world}",
            "data_generation": "AR(1) rows drawn in HBM per 100k-row block (torch Philox, "
                               "seeded per block: the same matrix at every world size)"}


# ---------------------------------------------------------------------------
# clocks (nvidia-smi sampled during the timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,"
              "clocks.mem,temperature.gpu,temperature.memory")

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
        time.sleep(0.3)

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
        mem, power, temp = [], [], []
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
            for dst, idx in ((power, 2), (mem, 8), (temp, 10)):
                try:
                    dst.append(float(parts[idx]))
                except (ValueError, IndexError):
                    pass
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm), "mem_mhz": statistics.median(mem) if mem else None,
                "power_w_max": max(power) if power else None,
                "mem_temp_c_max": max(temp) if temp else None}


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(key):
    """dram bytes (read + write) per launch of a kernel from the committed ncu
    --set full captures (profiles/ncu_summary.json), keyed by config/kernel."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        ks = d.get("kernels", {})
        v = ks.get(key)
        if v is None and key.startswith("C2/"):      # round-1 captures are keyed by kernel
            v = ks.get(key.split("/", 1)[1])
        return v.get("dram_bytes_per_launch") if v else None
    except Exception:
        return None


def kf_roofline(st, n, p, s_el, peak, peak_src, traffic_key):
    """HBM roofline of the single-pass kernel kf_fused_s from the per-launch
    CUDA-event durations (algorithmic bytes: X once + y, u_{t-1}, u_t, beta)."""
    avg = lambda k: st[k + "_ms"] / max(1, st[k + "_count"])
    kf_bytes = n * p * s_el + 8 * (4 * n + p)
    achieved = kf_bytes / (avg("k2") / 1e3) / 1e9
    return {"bound": "hbm", "kernel": "kf_fused_s", "achieved": achieved, "peak": peak,
            "unit": "GB/s", "frac": achieved / peak, "peak_source": peak_src,
            "frac_of_nominal_7700": achieved / 7700.0,
            "peak_note": ("the measured peak is a COPY (read + write) bandwidth; this kernel only "
                          "reads X, and a read-only stream can exceed the copy figure (frac > 1 is "
                          "not an error: see frac_of_nominal_7700 and the ncu DRAM traffic)"),
            "traffic": ncu_traffic(traffic_key), "algorithmic_bytes_per_launch": kf_bytes,
            "launch_ms": avg("k2"),
            "other_kernels": {"kr_reduce_epilogue": {"launch_ms": avg("k1")},
                              "k3_prox_window": {"launch_ms": avg("k3")}}}


# ---------------------------------------------------------------------------
# CPU baselines: the unmodified reference (baseline/_ref) and the oracle port
# ---------------------------------------------------------------------------
def _reference_module():
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "l0cert")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        import l0cert.fista as rf
        import l0cert.model as rm
        return rf, rm
    except Exception as exc:   # reported by the caller
        log(f"[bench] reference import failed: {exc!r}")
        return None


def time_reference(X, y, loss, k, M, lam2, L, iters, warm=2):
    """The reference's own solve_relaxation (fista.py:76-222), unmodified, on
    all host threads: K iterations after a warm-up solve (numba compile / cache
    load).  Returns seconds per iteration or None if the reference is absent."""
    mods = _reference_module()
    if mods is None:
        return None
    rf, rm = mods
    import threadpoolctl
    kind = {"squared_error": rm.LossKind.SQUARED_ERROR, "logistic": rm.LossKind.LOGISTIC}[loss]
    inst = rm.ProblemInstance(X=X, y=y, loss=kind, k=int(k), M=float(M), lambda2=float(lam2))
    with threadpoolctl.threadpool_limits(os.cpu_count()):
        rf.solve_relaxation(inst, opts=rf.FistaOptions(lipschitz=L, max_iterations=warm,
                                                       gap_tolerance=1e-300))
        t0 = time.perf_counter()
        rep = rf.solve_relaxation(inst, opts=rf.FistaOptions(lipschitz=L, max_iterations=iters,
                                                             gap_tolerance=1e-300))
        dt = time.perf_counter() - t0
    return dt / max(1, rep.iterations)


def time_port(X, y, loss, k, M, lam2, L, iters, warm=2):
    """The oracle port (numpy/OpenBLAS + C PAVA) on all host threads."""
    import threadpoolctl
    from oracle import l0_oracle
    with threadpoolctl.threadpool_limits(os.cpu_count()):
        l0_oracle.fista(X, y, loss, k, M, lam2, L=L, max_iter=warm, gap_tol=1e-300,
                        stop_on_gap=False)
        t0 = time.perf_counter()
        l0_oracle.fista(X, y, loss, k, M, lam2, L=L, max_iter=iters, gap_tol=1e-300,
                        stop_on_gap=False)
        dt = time.perf_counter() - t0
    return dt / iters


def cpu_baseline_c2(cd, iters, warm=2, prefer_reference=True):
    X = cd.X if cd.X.dtype == np.float64 else cd.X.astype(np.float64)
    cores = os.cpu_count()
    out = {"unit": "iters/s", "cores": cores}
    s_ref = time_reference(X, cd.y, cd.loss, cd.k, cd.M, cd.lambda2, L_C2, iters, warm) \
        if prefer_reference else None
    s_port = time_port(X, cd.y, cd.loss, cd.k, cd.M, cd.lambda2, L_C2, iters, warm)
    if s_ref is not None:
        out.update(value=1.0 / s_ref, kind="reference",
                   sample=f"{iters} FISTA iterations of C2 (after {warm} warm-up) with the "
                          f"unmodified reference l0cert.fista.solve_relaxation (baseline/_ref), "
                          f"{cores} threads", port_value=1.0 / s_port)
    else:
        out.update(value=1.0 / s_port, kind="port",
                   sample=f"{iters} FISTA iterations of C2 (after {warm} warm-up) with the "
                          f"numpy/OpenBLAS + C-PAVA oracle port, {cores} threads")
    return out


def c5_host_sample(rows, device):
    """The leading `rows` rows of C5 (generator block 0) copied to host fp64,
    with y: the bounded CPU sample whose per-iteration time scales with n."""
    from paper_2502_09502_b200 import data
    X, y = data.c5_shard_device(0, rows, device)
    return X.double().cpu().numpy(), y.cpu().numpy()


def cpu_baseline_c5(n_full, rows, iters, device, L=None):
    Xh, yh = c5_host_sample(rows, device)
    if L is None:
        import scipy.sparse.linalg as sla
        from scipy.sparse.linalg import LinearOperator
        op = LinearOperator((Xh.shape[1], Xh.shape[1]), matvec=lambda v: Xh.T @ (Xh @ v),
                            dtype=np.float64)
        L = 2.0 * 1.01 * float(sla.eigsh(op, k=1, which="LA", tol=1e-8,
                                         return_eigenvectors=False)[0])
    cores = os.cpu_count()
    s_ref = time_reference(Xh, yh, "squared_error", 25, 2.0, 0.1, L, iters, warm=1)
    s_port = time_port(Xh, yh, "squared_error", 25, 2.0, 0.1, L, iters, warm=1)
    s = s_ref if s_ref is not None else s_port
    scale = rows / n_full           # per-iteration work is linear in n at fixed p
    return {"value": scale / s, "unit": "iters/s", "cores": cores,
            "kind": "reference" if s_ref is not None else "port",
            "sample": f"{iters} FISTA iterations on the leading {rows} rows of C5 (fp64 on host), "
                      f"{'unmodified reference' if s_ref is not None else 'oracle port'}, "
                      f"{cores} threads; rate extrapolated x{rows}/{n_full} to the full n",
            "port_value": scale / s_port}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    if world > 1 and args.shard == "rows":
        import torch
        dev = "cuda" if torch.cuda.is_available() else "cpu"
        n = int(1_000_000 * args.c5_scale)
        cb = cpu_baseline_c5(n, args.c5_cpu_rows, max(1, min(args.steps, 5)), dev)
        cfg = c5_config(n, 10_000, world)
        dtype = "f64"
    else:
        cd = c2_inputs(args.scale)
        cb = cpu_baseline_c2(cd, args.steps, warm=min(args.warmup, 2))
        cfg = c2_config(cd)
        dtype = "f64"
    line = {"metric": METRIC, "value": cb["value"], "unit": "iters/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / cb["value"],
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": dtype, "data": "synthetic (seeded, see config)",
            "config": cfg, "impl": "reference", "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "iters/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# batched nodes (C4): tensor-core roofline
# ---------------------------------------------------------------------------
def tensor_peak():
    """Dense fp16 / bf16 tensor peak of this pool's B200s (MEASURED_PEAKS.json:
    cuBLAS bf16 8192^3, burst and sustained); kind::f16 runs at the bf16 rate."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return (float(d["bf16_tflops"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])),
                "measured (MEASURED_PEAKS.json bf16_tflops; kind::f16 has the bf16 rate)")
    except Exception:
        return 2250.0, 2250.0, "fallback (B200_PROFILING.md dense fp16 / bf16)"


def c4_setup(args, nodes_total):
    import paper_2502_09502_b200 as eng
    from paper_2502_09502_b200 import data
    t0 = time.time()
    cd = data.make_config("C4", scale=args.c4_scale, nodes=nodes_total)
    inst = eng.ProblemInstance(cd.X, cd.y, eng.LossKind.SQUARED_ERROR, cd.k, cd.M, cd.lambda2,
                               dtype="fp32")
    nodes = [None] + [eng.NodeState(fixed_one=f1, fixed_zero=f0)
                      for f0, f1 in cd.nodes[:nodes_total - 1]]
    L = eng.lipschitz_constant(inst, method="lanczos")
    log(f"[bench] C4 generated + L in {time.time() - t0:.1f}s")
    return cd, inst, nodes, L


def run_batched(args):
    """C4: 512 node relaxations (n=20000, p=5000 fp32) advanced together; the two
    X passes per iteration are tcgen05 3xTF32 contractions."""
    import torch
    import paper_2502_09502_b200 as eng
    cd, inst, nodes, L = c4_setup(args, args.c4_nodes)
    B, n, p, K = len(nodes), cd.n, cd.p, args.c4_steps
    opts = lambda it, prof: eng.FistaOptions(lipschitz=L, max_iterations=it, stop_on_gap=False,
                                             profile=prof)
    eng.solve_relaxation_batched(inst, nodes, opts=opts(3, False))
    eng.solve_relaxation_batched(inst, nodes, opts=opts(3, True))
    torch.cuda.synchronize()
    clocks = ClockSampler(0)
    clocks.start()
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
    useful_t = 2.0 * n * p * B * (1.0 + checks)
    burst, sustained, peak_src = tensor_peak()
    tensor_t = 3 * useful_t / (gt / 1e3) / 1e12
    cpu = None
    if not args.no_cpu:
        X64 = cd.X.astype(np.float64)
        nd = nodes[1]
        import threadpoolctl
        from oracle import l0_oracle
        cores = os.cpu_count()
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
            "contraction": "tcgen05 kind::f16, 3xFP16 (power-of-two scaled hi/lo split), fp32 TMEM "
                           "accumulation; the forward contraction only over the X columns of the "
                           "nodes' step supports (slot cache)",
            "roofline": {"bound": "tensor", "unit": "TFLOP/s",
                         "kernel": "tc_gemm_kernel (transpose X^T [R | Z], the dominant contraction)",
                         "achieved": tensor_t, "peak": burst, "frac": tensor_t / burst,
                         "peak_source": peak_src, "peak_sustained": sustained,
                         "frac_vs_sustained": tensor_t / sustained,
                         "flops_per_transpose_launch": 3 * useful_t,
                         "note": "tensor FLOPs count the 3 fp16 products of the hi/lo split; "
                                 "X^T [R | Z] has 2 n p B flops per product (x2 rows on bound "
                                 "checks, averaged over the iterations)"},
            "ms_per_iteration_split": {"gemm_transpose": gt, "prox": px, "gemm_forward": gf},
            "cpu_baseline": cpu}


# ---------------------------------------------------------------------------
# C5 on one GPU (the row-sharding config at N=1)
# ---------------------------------------------------------------------------
def run_c5_single(args):
    import torch
    import paper_2502_09502_b200 as eng
    from paper_2502_09502_b200 import data
    n, p = int(data.C5_N * args.c5_scale), data.C5_P
    t0 = time.time()
    X, y = data.c5_shard_device(0, n, torch.device("cuda", 0), n=n)
    inst = eng.ProblemInstance(X, y.cpu().numpy(), eng.LossKind.SQUARED_ERROR, 25, 2.0, 0.1,
                               dtype="fp32")
    inst.device_problem()
    torch.cuda.synchronize()
    gen_s = time.time() - t0
    t0 = time.time()
    L = eng.lipschitz_constant(inst, method="lanczos")
    l_s = time.time() - t0
    log(f"[bench] C5 n={n} generated in {gen_s:.1f}s, Lanczos L={L:.6g} in {l_s:.1f}s")
    K = args.c5_steps
    o = lambda k, prof: eng.FistaOptions(lipschitz=L, max_iterations=k, gap_tolerance=1e-300,
                                         stop_on_gap=False, profile=prof)
    eng.solve_relaxation(inst, opts=o(3, False), return_device=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rep = eng.solve_relaxation(inst, opts=o(K, False), return_device=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    assert rep.iterations == K
    st = eng.solve_relaxation(inst, opts=o(K, True), return_device=True).stats
    peak, src = measured_peak()
    roof = kf_roofline(st, n, p, 4, peak, src, "C5/kf_fused_s") if st.get("single_pass") else None
    f32 = fp32_mode_run(eng, inst, L, K, n, p, peak, src)
    cpu = None
    if not args.no_cpu:
        cpu = cpu_baseline_c5(n, args.c5_cpu_rows, 3, "cuda", L=L)
    del inst, X
    torch.cuda.empty_cache()
    return {"workload": C5_WORKLOAD.split(";")[0] + "; one GPU", "n": n, "p": p,
            "value": K / (ms / 1e3), "unit": "iters/s", "steps": K, "ms_per_step": ms / K,
            "engine_path": "single_pass" if st.get("single_pass") else "two_pass",
            "cluster_size": st.get("cluster_size"), "lipschitz": L, "lipschitz_method": "lanczos",
            "setup_s": {"generate": gen_s, "lanczos": l_s}, "roofline": roof, "cpu_baseline": cpu,
            "restarts": rep.restarts, "primal": rep.primal_value, "dual": rep.dual_bound,
            "fp32_mode": f32}


def fp32_mode_run(eng, inst, L, K, n, p, peak, src):
    """The same K iterations in the fp32 mode (FistaOptions.fp32_forward: X beta
    in fp32 products, fp64 reductions -- BASELINE's "fp32 X with fp64
    reductions", north-star tolerance 1e-5; tests/test_gpu_fullsize.py)."""
    import torch
    o = lambda k, prof: eng.FistaOptions(lipschitz=L, max_iterations=k, gap_tolerance=1e-300,
                                         stop_on_gap=False, profile=prof, fp32_forward=True)
    eng.solve_relaxation(inst, opts=o(3, False), return_device=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rep = eng.solve_relaxation(inst, opts=o(K, False), return_device=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    st = eng.solve_relaxation(inst, opts=o(K, True), return_device=True).stats
    roof = kf_roofline(st, n, p, 4, peak, src, "none") if st.get("single_pass") else None
    return {"value": K / (ms / 1e3), "unit": "iters/s", "ms_per_step": ms / K, "roofline": roof,
            "primal": rep.primal_value, "dual": rep.dual_bound, "restarts": rep.restarts,
            "arithmetic": "X beta: fp32 products, fp64 reductions; X^T r and everything else fp64"}


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
    L = eng.lipschitz_constant(inst, method="lanczos")
    gen_s = time.time() - t0
    o = lambda k, prof: eng.FistaOptions(lipschitz=L, max_iterations=k, gap_tolerance=1e-300,
                                         stop_on_gap=False, profile=prof)
    eng.solve_relaxation(inst, opts=o(5, False), return_device=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t_host = time.perf_counter()
    rep = eng.solve_relaxation(inst, opts=o(iters, False), return_device=True)
    e1.record()
    torch.cuda.synchronize()
    wall_ms = (time.perf_counter() - t_host) * 1e3
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
        if cd.loss != "squared_error" and cd.dtype == "fp32":
            # SPEC kernel: KF accumulates the no-restart candidate only; restart and
            # bound-check iterations add one K2 transpose pass behind KR
            kern["kr_reduce_plus_conditional_k2"] = kern.pop("kr_reduce")
            kern["kr_reduce_plus_conditional_k2"]["note"] = (
                "average over all iterations of KR plus the K2 pass that runs on restart "
                "iterations only (one extra read of X on those)")
            kern["kf_fused_s"]["variant"] = (
                "SPEC: the no-restart candidate (one accumulated vector), plus X^T zeta in a "
                "two-vector kernel on bound-check iterations; both kernels are launched every "
                "iteration inside the timed event pair and one returns at entry, so launch_ms "
                "averages the two")
        elif cd.loss == "squared_error":
            kern["kf_fused_s"]["variant"] = "LIN (one accumulated vector, candidates by linearity)"
    else:
        kern = {"k1_forward": {"launch_ms": avg("k1"), "achieved_gbs": (xb + 8 * (p + 2 * n)) / avg("k1") / 1e6},
                "k2_transpose": {"launch_ms": avg("k2"), "achieved_gbs": (xb + 8 * (3 * n + 5 * p)) / avg("k2") / 1e6},
                "k3_prox_window": {"launch_ms": avg("k3")}}
        for k in ("k1_forward", "k2_transpose"):
            kern[k]["frac"] = kern[k]["achieved_gbs"] / peak
    out = {"config": name, "n": n, "p": p, "dtype": cd.dtype, "loss": cd.loss, "k": cd.k, "M": cd.M,
           "lambda2": cd.lambda2, "lipschitz": L, "lipschitz_method": "lanczos", "iterations": iters,
           "value": iters / (ms / 1e3), "unit": "iters/s", "ms_per_iteration": ms / iters,
           "engine_path": "single_pass" if st.get("single_pass") else "two_pass",
           "x_bytes": xb, "l2_resident": xb < 100e6, "kernels": kern, "peak_gbs": peak,
           "primal": rep.primal_value, "dual": rep.dual_bound, "restarts": rep.restarts,
           "gpu_launches": rep.stats.get("gpu_launches"),
           "prox_full_passes": rep.stats.get("prox_full_passes"), "host_wall_ms": wall_ms,
           "setup_s": gen_s}
    if cd.dtype == "fp32" and st.get("single_pass"):
        src = measured_peak()[1]
        out["fp32_mode"] = fp32_mode_run(eng, inst, L, iters, n, p, peak, src)
    del inst
    torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------------------
# ours, N = 1
# ---------------------------------------------------------------------------
def e2e_solves(eng, cd, make_x, solves, engine):
    """Full solves to the C2 target through the public API from host X."""
    import torch
    iters, secs, reps = 0, 0.0, []
    for i in range(solves + 1):
        warm = i == 0          # one untimed warm-up call (process-level one-time costs)
        X = make_x()
        inst_h = eng.ProblemInstance(X, cd.y, eng.LossKind.SQUARED_ERROR, cd.k, cd.M, cd.lambda2)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = eng.solve_relaxation(inst_h, opts=eng.FistaOptions(
            lipschitz=L_C2, gap_tolerance=1e-300, gap_tolerance_rel=REL_GAP, engine_path=engine))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if not warm:
            iters += r.iterations
            secs += dt
        reps.append({"iterations": r.iterations, "seconds": dt, "rel_gap": r.gap / abs(r.primal_value),
                     "termination": r.termination.value, "warmup": warm})
        inst_h.release_device()
        del inst_h
    return (iters / secs if secs > 0 else None), reps


def run_ours(args):
    import torch
    world, rank, local = dist_env()
    if world > 1 or args.force_dist:
        return run_ours_sharded(args, world, rank, local)
    torch.cuda.set_device(0)
    import paper_2502_09502_b200 as eng
    eng.native.load()
    cd = c2_inputs(args.scale)
    inst = eng.ProblemInstance(cd.X, cd.y, eng.LossKind.SQUARED_ERROR, cd.k, cd.M, cd.lambda2)
    t0 = time.time()
    inst.device_problem()
    torch.cuda.synchronize()
    log(f"[bench] upload {time.time() - t0:.2f}s")
    K, W = args.steps, args.warmup

    def fixed(iters, profile):
        return eng.FistaOptions(lipschitz=L_C2, max_iterations=iters, gap_tolerance=1e-300,
                                stop_on_gap=False, profile=profile, engine_path=args.engine)

    # warm-up: W iterations with the same options as the timed run (graph
    # capture, caches), then the profiled variant (its graphs are kept apart)
    eng.solve_relaxation(inst, opts=fixed(W, False), return_device=True)
    eng.solve_relaxation(inst, opts=fixed(W, True), return_device=True)
    # ... and one untimed solve of the timed length: the engine captures one CUDA
    # graph per replay length, and a K-iteration solve is a single replay of K + 1
    # iterations, so without this the timed call would include its graph capture
    eng.solve_relaxation(inst, opts=fixed(K, False), return_device=True)
    eng.solve_relaxation(inst, opts=fixed(K, True), return_device=True)
    torch.cuda.synchronize()
    # timed region: exactly K iterations, CUDA events, clocks sampled
    clocks = ClockSampler(0)
    clocks.start()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    start.record()
    rep = eng.solve_relaxation(inst, opts=fixed(K, False), return_device=True)
    end.record()
    torch.cuda.synchronize()
    ms = start.elapsed_time(end)
    assert rep.iterations == K, rep.iterations
    value = K / (ms / 1e3)
    launches = int(rep.stats["gpu_launches"])
    # the same K iterations again with CUDA events around every kernel inside the
    # graphs (on the engine's stream): the per-launch durations behind the
    # roofline.  The events add ~10 us of graph nodes per iteration, so the
    # headline value above comes from the un-instrumented run.
    start.record()
    rep_p = eng.solve_relaxation(inst, opts=fixed(K, True), return_device=True)
    end.record()
    torch.cuda.synchronize()
    ms_prof = start.elapsed_time(end)
    clk = clocks.stop()
    st = rep_p.stats
    log(f"[bench] {K} its in {ms:.2f} ms -> {value:.1f} it/s; k1 {st['k1_ms'] / max(1, st['k1_count']):.4f} "
        f"ms k2 {st['k2_ms'] / max(1, st['k2_count']):.4f} ms k3 {st['k3_ms'] / max(1, st['k3_count']):.4f} ms")
    peak, peak_src = measured_peak()
    n, p = cd.n, cd.p
    single = bool(st.get("single_pass"))
    if single:
        roofline = kf_roofline(st, n, p, 8, peak, peak_src, "C2/kf_fused_s")
    else:
        avg = lambda k: st[k + "_ms"] / max(1, st[k + "_count"])
        k2_bytes = n * p * 8 + 8 * (3 * n + 5 * p)
        achieved = k2_bytes / (avg("k2") / 1e3) / 1e9
        roofline = {"bound": "hbm", "kernel": "k2_transpose", "achieved": achieved, "peak": peak,
                    "unit": "GB/s", "frac": achieved / peak, "peak_source": peak_src,
                    "traffic": ncu_traffic("C2/k2_transpose"),
                    "algorithmic_bytes_per_launch": k2_bytes, "launch_ms": avg("k2")}
    roofline.update({
        "launch_ms_source": "CUDA events around each kernel inside the graphs (engine stream), "
                            "second run of the same K iterations (instrumented ms/step %.4f)" % (ms_prof / K),
        "engine": "single pass (X read once per iteration)" if single else "two pass",
        "iteration_bytes_2pass": 2 * n * p * 8,
        "iteration_rate_vs_2pass_roofline": (2 * n * p * 8) / (ms / 1e3 / K) / 1e9 / peak,
        "note": "iteration_rate_vs_2pass_roofline > 1 is possible only because the single-pass "
                "engine reads X once per iteration" if single else ""})
    # end to end through the public API with host-resident X: numpy (pageable,
    # the drop-in call) is the headline; a pinned torch tensor is reported beside
    h2d = cd.X.nbytes + cd.y.nbytes
    d2h = cd.p * 8
    e2e_np, reps_np = e2e_solves(eng, cd, lambda: cd.X, args.e2e_solves, args.engine)
    Xpin = torch.from_numpy(cd.X).pin_memory()
    e2e_pin, reps_pin = e2e_solves(eng, cd, lambda: Xpin, args.e2e_solves, args.engine)
    del Xpin
    e2e = {"value": e2e_np, "unit": "iters/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
           "step": "one solve_relaxation call to relative gap 1e-6 from a host numpy X (pageable; "
                   "staged by the engine's multi-threaded pinned ring, l0_upload_rows)",
           "solves": reps_np, "pinned_tensor_value": e2e_pin, "pinned_tensor_solves": reps_pin}
    log(f"[bench] e2e numpy {e2e_np} it/s, pinned {e2e_pin} it/s")
    cb = cpu_baseline_c2(cd, args.cpu_iters) if not args.no_cpu else None
    del inst
    torch.cuda.empty_cache()
    sections = {}
    if args.c5_steps > 0:
        try:
            sections["c5"] = run_c5_single(args)
            log(f"[bench] C5 {sections['c5']['value']:.1f} it/s")
        except Exception as exc:   # reported, never silently dropped
            sections["c5"] = {"error": repr(exc)}
    batched = None
    if args.c4_nodes > 0:
        try:
            batched = run_batched(args)
            log(f"[bench] C4 {batched['value']:.0f} node-it/s {batched['ms_per_iteration_split']}")
        except Exception as exc:
            batched = {"error": repr(exc)}
    others = []
    for name in [c for c in args.configs.split(",") if c and c != "none"]:
        try:
            others.append(run_config(name, args.config_steps))
            log(f"[bench] {name} {others[-1]['value']:.1f} it/s {others[-1]['kernels']}")
        except Exception as exc:
            others.append({"config": name, "error": repr(exc)})
    line = {"metric": METRIC,
            "value": value, "unit": "iters/s", "n_gpus": 1, "steps": K, "warmup": W,
            "ms_per_step": ms / K, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference generator, seed 0)",
            "config": c2_config(cd), "roofline": roofline, "cpu_baseline": cb, "e2e": e2e,
            "gpu_launches": launches, "clocks": clk,
            "warmup_detail": (f"one {W}-iteration solve (the W warm-up steps) and one {K}-iteration "
                              "solve, both untimed: the engine keeps one CUDA graph per replay "
                              "length, so the timed call re-uses a captured graph as any second "
                              "call with the same options does"),
            "engine_path": "single_pass" if single else "two_pass",
            "restarts": rep.restarts, "final_gap": rep.gap,
            "prox_full_passes": st.get("prox_full_passes"), "topk_fallbacks": st.get("topk_fallbacks"),
            "c5_single_gpu": sections.get("c5"), "batched_nodes": batched, "other_configs": others}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# ours, N > 1
# ---------------------------------------------------------------------------
def run_ours_sharded(args, world, rank, local):
    """--shard rows (default): C5's rows over the ranks, each rank generating
    its own rows in HBM; the engine all-reduces [X_r^T r | X_r^T zeta | F*]
    and the loss over NCCL inside its CUDA graphs every iteration ("strong").
    --shard nodes: C4's 512 nodes over the ranks, one batched call per rank on
    its share (no collective).  value = all ranks' units / max-over-ranks
    device time."""
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2502_09502_b200 import distributed as shard
    import paper_2502_09502_b200 as eng
    from paper_2502_09502_b200 import data
    eng.native.load()
    K, W = args.steps, args.warmup
    dev = torch.device("cuda", local)
    red = lambda t: dist.all_reduce(t)
    e2e = None
    if args.shard == "rows":
        n, p = int(data.C5_N * args.c5_scale), data.C5_P
        r0, r1 = shard.row_range(n, world, rank)
        t0 = time.time()
        X, y = data.c5_shard_device(r0, r1, dev, n=n, allreduce=red)
        sp = shard.ShardedProblem(X, y.cpu().numpy(), eng.LossKind.SQUARED_ERROR, 25, 2.0, 0.1,
                                  n_global=n, dtype="fp32")
        L = sp.lipschitz(method="lanczos")
        log(f"[bench] rank {rank}: rows [{r0}, {r1}) generated + L={L:.6g} in {time.time() - t0:.1f}s")
        opts = lambda it: eng.FistaOptions(lipschitz=L, max_iterations=it, gap_tolerance=1e-300,
                                           stop_on_gap=False)
        solve = lambda it: shard.solve_relaxation_sharded(sp, opts=opts(it))
        units, cfg, unit_name = 1, c5_config(n, p, world), "iters/s"
    else:
        cd, inst, nodes, L = c4_setup(args, args.c4_nodes)
        mine = shard.shard_nodes(nodes, world, rank)
        my_nodes = [nodes[i] for i in mine]
        opts = lambda it: eng.FistaOptions(lipschitz=L, max_iterations=it, stop_on_gap=False)
        solve = lambda it: eng.solve_relaxation_batched(inst, my_nodes, opts=opts(it),
                                                        return_device=True)[0]
        units, unit_name = len(nodes), "node-iters/s"
        cfg = {"workload": f"C4: {len(nodes)} node relaxations (n={cd.n}, p={cd.p} fp32) split over "
                           f"the GPUs, one batched tcgen05 call per rank", "nodes": len(nodes),
               "parallelism": f"nodes{world}"}
    solve(W)
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local) if rank == 0 else None
    if clocks:
        clocks.start()
    start.record()
    rep = solve(K)
    end.record()
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop() if clocks else None
    ms = torch.tensor([start.elapsed_time(end)], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    launches = torch.tensor([float(rep.stats["gpu_launches"])], device=dev)
    dist.all_reduce(launches)
    if args.shard == "rows" and args.e2e_solves > 0:
        # end to end: this rank's rows from pinned host memory, uploaded and
        # solved K iterations per call (H2D of X_r, y_r and D2H of beta inside)
        Xh = X.cpu().pin_memory()
        yh = y.cpu().numpy()
        del sp
        torch.cuda.empty_cache()
        dist.barrier()
        t0 = time.perf_counter()
        sp2 = shard.ShardedProblem(Xh, yh, eng.LossKind.SQUARED_ERROR, 25, 2.0, 0.1,
                                   n_global=n, dtype="fp32")
        r2 = shard.solve_relaxation_sharded(sp2, opts=opts(K))
        torch.cuda.synchronize()
        dt = torch.tensor([time.perf_counter() - t0], device=dev)
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        e2e = {"value": K / float(dt.item()), "unit": "iters/s",
               "h2d_bytes_per_step": int(Xh.numel() * 4 + yh.size * 8) * world,
               "d2h_bytes_per_step": int(p * 8) * world,
               "step": f"per rank: its C5 rows from pinned host memory -> ShardedProblem + "
                       f"{K}-iteration solve (max over ranks, host wall clock)"}
    if rank == 0:
        line = {"metric": METRIC if args.shard == "rows" else
                "node FISTA iterations/s (C4 nodes sharded over the GPUs)",
                "value": units * K / (ms / 1e3), "unit": unit_name, "n_gpus": world,
                "steps": K, "warmup": W, "ms_per_step": ms / K, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None,
                "dtype": "f32 X / f64 arithmetic", "data": "synthetic (seeded, see config)",
                "config": cfg, "gpu_launches": int(launches.item()), "clocks": clk, "e2e": e2e,
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
    ap.add_argument("--shard", default="rows", choices=["rows", "nodes"],
                    help="N > 1: C5 rows over the GPUs (default) or C4 nodes over the GPUs")
    ap.add_argument("--c5-steps", type=int, default=100, help="C5 section at N=1 (0: skip)")
    ap.add_argument("--c5-scale", type=float, default=1.0, help="shrink C5's n (testing only)")
    ap.add_argument("--c5-cpu-rows", type=int, default=20000)
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
