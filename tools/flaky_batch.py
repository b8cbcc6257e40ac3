import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np
from test_gpu_batch import _c4_instance
from paper_2502_09502_b200 import FistaOptions, lipschitz_constant, solve_relaxation, solve_relaxation_batched
inst, nodes = _c4_instance(0.1, 8)
L = lipschitz_constant(inst)
print("L", repr(L))
for tol in (1e-4, 1e-3):
    for rep in range(3):
        opts = FistaOptions(max_iterations=3000, lipschitz=L, gap_tolerance=tol)
        reps = solve_relaxation_batched(inst, nodes, opts=opts)
        refs = [solve_relaxation(inst, nd, opts=opts) for nd in nodes]
        print(tol, rep, [r.iterations for r in reps], [r.iterations for r in refs], "obj", refs[0].primal_value,
              [f"{r.gap:.2e}" for r in reps])
