"""Per-step timing of the solve sweep program (CUDA events, each step repeated alone)."""
import argparse
import sys

sys.path.insert(0, ".")
import torch

import bench
from paper_1612_02736_b200 import _ext, build_stage
from paper_1612_02736_b200.geometry import enumerate_gauss_nodes

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--nrhs", type=int, default=1)
args = ap.parse_args()
tree, spec, p, q, desc = bench.make_config(args.config, 0)
plan = enumerate_gauss_nodes(tree, q)
solver = build_stage(tree, spec, p, q, plan=plan)
nl, m = solver._n_leaves, (p - 2) ** 2
g = torch.ones((nl * m, args.nrhs), dtype=torch.float64, device="cuda")
f = torch.ones((plan.node[tree.root].ext.size, args.nrhs), dtype=torch.float64, device="cuda")
solver.solve_device(f, g)
prog = solver._program(args.nrhs)
lib = _ext.load()
s = torch.cuda.current_stream().cuda_stream
tot = 0.0
totb = 0.0
for name, steps in (("up", prog["up"]), ("down", prog["down"])):
    for st in steps:
        reps = 20
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        lib.hps_sweep_gemv(st, s)
        e0.record()
        for _ in range(reps):
            lib.hps_sweep_gemv(st, s)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / reps * 1e3
        byt = 8.0 * st.nitems * (st.R * st.K + (st.R2 * st.K2 if st.mode2 else 0))
        if st.A2.stride == 0 and st.mode2:
            byt -= 8.0 * st.nitems * st.R2 * st.K2
        if st.A.stride == 0:
            byt = 8.0 * st.R * st.K
        tot += us
        totb += byt
        print(f"{name:4s} items={st.nitems:6d} R={st.R:5d} K={st.K:5d} mode2={st.mode2} R2={st.R2:5d} K2={st.K2:5d} "
              f"{us:8.1f} us  {byt / us / 1e3:7.1f} GB/s")
print(f"sum {tot:.1f} us, {totb / 1e9:.3f} GB, {totb / tot / 1e3:.1f} GB/s")
