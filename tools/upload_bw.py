"""Host -> HBM upload of C2's X (2.05 GB fp64): pinned torch copy vs the
engine's pageable staging path (l0_upload_rows) under L0_UPLOAD_MB /
L0_UPLOAD_THREADS settings.  python tools/upload_bw.py"""
import os, subprocess, sys, time
sys.path.insert(0, ".")
import numpy as np
import torch

if len(sys.argv) > 1 and sys.argv[1] == "child":
    import paper_2502_09502_b200 as eng
    from paper_2502_09502_b200 import native, _device
    n = p = 16000
    X = np.random.default_rng(0).standard_normal((n, p))
    Xt = torch.from_numpy(X)
    Xd = torch.empty((n, p), dtype=torch.float64, device="cuda")
    lib = native.load()
    best = 1e9
    for _ in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        native.check(lib.l0_upload_rows(Xd.data_ptr(), p * 8, Xt.data_ptr(), p * 8, p * 8, n, 16,
                                        _device.stream_handle()))
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    assert torch.equal(Xd[::997].cpu(), Xt[::997])
    print(f"staging MB={os.environ.get('L0_UPLOAD_MB','32')} T={os.environ.get('L0_UPLOAD_THREADS','16')}: "
          f"{X.nbytes / best / 1e9:.1f} GB/s ({best*1e3:.1f} ms)", flush=True)
    sys.exit(0)

n = p = 16000
Xp = torch.empty((n, p), dtype=torch.float64).pin_memory()
Xp.normal_()
Xd = torch.empty((n, p), dtype=torch.float64, device="cuda")
best = 1e9
for _ in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    Xd.copy_(Xp, non_blocking=True)
    torch.cuda.synchronize()
    best = min(best, time.perf_counter() - t0)
print(f"pinned torch copy: {Xp.numel() * 8 / best / 1e9:.1f} GB/s", flush=True)
del Xp, Xd
for mb in (1, 2, 4, 8, 16):
    for th in (4, 8, 12, 16):
        env = dict(os.environ, L0_UPLOAD_MB=str(mb), L0_UPLOAD_THREADS=str(th))
        subprocess.run([sys.executable, __file__, "child"], env=env)
