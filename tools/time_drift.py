"""C2 iteration time over back-to-back 400-iteration solves with nvidia-smi clocks,
temperatures and power after each (run-to-run drift under sustained load)."""
import sys, time
sys.path.insert(0, ".")
import torch, subprocess
import paper_2502_09502_b200 as eng
from paper_2502_09502_b200 import data
cd = data.make_config("C2", scale=1.0)
inst = eng.ProblemInstance(cd.X, cd.y, eng.LossKind.SQUARED_ERROR, cd.k, cd.M, cd.lambda2)
o = lambda k: eng.FistaOptions(lipschitz=2.9908e5, max_iterations=k, gap_tolerance=1e-300, stop_on_gap=False)
eng.solve_relaxation(inst, opts=o(5), return_device=True)
for i in range(8):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); eng.solve_relaxation(inst, opts=o(400), return_device=True); b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    q = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,temperature.gpu,temperature.memory,power.draw", "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
    print(f"solve {i}: {ms/400*1e3:.1f} us/it  [{q}]", flush=True)
