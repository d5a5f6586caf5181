"""Run one sweep step of a config's solve program repeatedly (for ncu): --which last|first|index."""
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
ap.add_argument("--pass_", default="down")
ap.add_argument("--index", type=int, default=-1)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
tree, spec, p, q, desc = bench.make_config(args.config, 0)
solver = build_stage(tree, spec, p, q, plan=enumerate_gauss_nodes(tree, q))
nl, m = solver._n_leaves, (p - 2) ** 2
g = torch.ones((nl * m, args.nrhs), dtype=torch.float64, device="cuda")
f = torch.ones((solver.plan.node[tree.root].ext.size, args.nrhs), dtype=torch.float64, device="cuda")
solver._program(args.nrhs)
torch.cuda.synchronize()
st = solver._program(args.nrhs)[args.pass_][args.index]
lib = _ext.load()
for _ in range(args.reps):
    lib.hps_sweep_gemv(st, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("done")
