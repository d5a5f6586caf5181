"""Config 5 end to end on the GPU: build (I/dt - Lap), then the full backward-Euler trajectory
(1000 steps x 16 RHS, device resident) — prints one JSON line."""
import argparse
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_1612_02736_b200 import build_stage, build_uniform_tree, problems
from paper_1612_02736_b200.geometry import count_chebyshev_dofs, enumerate_gauss_nodes
from paper_1612_02736_b200.timestepping import _leaf_points, be_run

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=128)
ap.add_argument("--steps", type=int, default=1000)
ap.add_argument("--nrhs", type=int, default=16)
args = ap.parse_args()
dt = 1e-3
tree = build_uniform_tree((0.0, 1.0, 0.0, 1.0), args.n)
plan = enumerate_gauss_nodes(tree, 15)
build_stage(tree, problems.config5_spec(dt), 16, 15, plan=plan)  # warm
torch.cuda.synchronize()
t0 = time.perf_counter()
solver = build_stage(tree, problems.config5_spec(dt), 16, 15, plan=plan)
torch.cuda.synchronize()
build_s = time.perf_counter() - t0
pts = _leaf_points(solver)
u0 = np.stack([problems.config5_initial(r)(pts.reshape(-1, 2)).reshape(solver._n_leaves, -1)
               for r in range(args.nrhs)], axis=-1)
u0 = torch.as_tensor(u0, device="cuda")
bpts = solver.plan.coords[solver.plan.node[tree.root].ext]
base = torch.as_tensor(bpts[:, 0] * (1.0 - bpts[:, 1]), device="cuda")[:, None].expand(-1, args.nrhs).contiguous()
fbuf = torch.empty_like(base)


def dirichlet(t):
    torch.mul(base, float(np.sin(2.0 * np.pi * t)), out=fbuf)
    return fbuf


be_run(solver, u0, dirichlet, dt, 3)  # warm (graph capture)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
st = be_run(solver, u0, dirichlet, dt, args.steps)
e1.record()
torch.cuda.synchronize()
sec = e0.elapsed_time(e1) / 1e3
ncheb = count_chebyshev_dofs(tree, 16)
u = st.leaf_tabulations()
print(json.dumps({"workload": f"config5 BE {args.n}x{args.n} p=16, {args.steps} steps x {args.nrhs} RHS",
                  "build_s": round(build_s, 4), "trajectory_s": round(sec, 4),
                  "ms_per_step": round(sec / args.steps * 1e3, 4),
                  "Mpts_per_s_per_rhs": round(ncheb * args.nrhs * args.steps / sec / 1e6, 1),
                  "finite": bool(torch.isfinite(u).all()), "max_abs_u": float(u.abs().max())}))
