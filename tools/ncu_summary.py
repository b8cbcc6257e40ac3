"""Build profiles/ncu_summary.json from ncu --set full reports:
python tools/ncu_summary.py out.json [CFG=]rep1.ncu-rep [[CFG=]rep2 ...]
(CFG= prefixes the kernel keys, e.g. C2=prof.ncu-rep -> "C2/kf_fused_s")"""
import csv, json, re, subprocess, sys

SHORT = [("kf_fused_s", "kf_fused_s"), ("kf_fused", "kf_fused"), ("k1_forward", "k1_forward"), ("k2_transpose", "k2_transpose"),
         ("k3_prox_window", "k3_prox_window"), ("kr_reduce", "kr_reduce"), ("tc_gemm_kernel", "tc_gemm_kernel"),
         ("kb_window", "kb_window"), ("kb_step", "kb_step"), ("kb_obj", "kb_obj"), ("kb_rhs", "kb_rhs"),
         ("k_mrhs", "k_mrhs"), ("k_std_stats", "k_std_stats")]
METRICS = {"gpu__time_duration.sum": ("duration_us", 1.0), "dram__bytes_read.sum": ("dram_read_bytes", None),
           "dram__bytes_write.sum": ("dram_write_bytes", None),
           "dram__throughput.avg.pct_of_peak_sustained_elapsed": ("dram_pct_of_ncu_peak", 1.0),
           "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active": ("tensor_pipe_pct", 1.0),
           "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active": ("tc_inst_pct", 1.0),
           "lts__t_sector_hit_rate.pct": ("l2_hit_pct", 1.0),
           "smsp__issue_active.avg.pct_of_peak_sustained_active": ("issue_active_pct", 1.0),
           "sm__warps_active.avg.pct_of_peak_sustained_active": ("warps_active_pct", 1.0),
           "launch__registers_per_thread": ("registers", 1.0), "launch__grid_size": ("grid", 1.0),
           "launch__block_size": ("block", 1.0)}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1.0, "ms": 1e3, "ns": 1e-3}
out = {"source": "ncu --set full --clock-control none (B200), tools/profile_round.sh", "kernels": {}}
for arg in sys.argv[2:]:
    cfg, rep = arg.split("=", 1) if "=" in arg else ("", arg)
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    if len(rows) < 3:
        continue
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        name = v[h.index("Kernel Name")]
        short = next((s for k, s in SHORT if k in name), None)
        if short is None:
            continue
        if cfg:
            short = f"{cfg}/{short}"
        rec = {"name": name, "report": rep}
        for m, (key, _) in METRICS.items():
            if m in h:
                i = h.index(m)
                try:
                    val = float(v[i].replace(",", ""))
                except ValueError:
                    continue
                rec[key] = val * UNIT.get(u[i], 1.0)
        rec["dram_bytes_per_launch"] = rec.get("dram_read_bytes", 0) + rec.get("dram_write_bytes", 0)
        prev = out["kernels"].get(short)
        # keep the longest launch of each kernel (early-exit launches are ~us)
        if prev is None or rec.get("duration_us", 0) > prev.get("duration_us", 0):
            out["kernels"][short] = rec
json.dump(out, open(sys.argv[1], "w"), indent=1)
print(json.dumps({k: (round(v.get("duration_us", 0), 1), v.get("dram_bytes_per_launch")) for k, v in out["kernels"].items()}))
