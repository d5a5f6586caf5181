"""Small driver for ncu launch lists: one build + a few eager solves of a config."""
import argparse
import sys

sys.path.insert(0, ".")
import torch

import bench
from paper_1612_02736_b200 import build_stage
from paper_1612_02736_b200.geometry import enumerate_gauss_nodes

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--nrhs", type=int, default=1)
ap.add_argument("--solves", type=int, default=2)
ap.add_argument("--builds", type=int, default=1)
args = ap.parse_args()
tree, spec, p, q, desc = bench.make_config(args.config, args.n)
plan = enumerate_gauss_nodes(tree, q)
for _ in range(args.builds):
    solver = build_stage(tree, spec, p, q, plan=plan)
torch.cuda.synchronize()
solver.use_graphs = False
nl, m = solver._n_leaves, (p - 2) ** 2
g = torch.ones((nl * m, args.nrhs), dtype=torch.float64, device="cuda")
f = torch.ones((plan.node[tree.root].ext.size, args.nrhs), dtype=torch.float64, device="cuda")
for _ in range(args.solves):
    solver.solve_device(f, g)
torch.cuda.synchronize()
print("done", desc)
