"""Where the host-API solve time goes (config 2): H2D of g/f, device solve, D2H of the results."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import bench
from paper_1612_02736_b200 import build_stage
from paper_1612_02736_b200.geometry import enumerate_gauss_nodes

tree, spec, p, q, desc = bench.make_config(int(sys.argv[1]) if len(sys.argv) > 1 else 2, 0)
solver = build_stage(tree, spec, p, q, plan=enumerate_gauss_nodes(tree, q))
g = solver._leaf_table(None)
gd = {int(n): g[r] for r, n in enumerate(solver._leaf_ids)}
f = solver._dirichlet(None)
for _ in range(3):
    solver.solve(f=f, g=g)
torch.cuda.synchronize()


def tm(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


prog = solver._program(1)
pool = prog["pool"]
lay = solver._layout
nl, m, P, N = solver._n_leaves, (p - 2) ** 2, p * p, solver.plan.n_gauss
gdev = pool[lay["G"]:lay["G"] + nl * m, 0]
gt = torch.as_tensor(g).reshape(-1)
gpin = gt.pin_memory()
print("full solve (host API)     %.3f ms" % tm(lambda: solver.solve(f=f, g=g)))
print("full solve (dict g)       %.3f ms" % tm(lambda: solver.solve(f=f, g=gd)))
stage = np.empty((nl, m))
print("dict -> table (concat)    %.3f ms" % tm(lambda: solver._leaf_table(gd, out=stage)))
print("H2D g pageable            %.3f ms  (%.1f MB)" % (tm(lambda: gdev.copy_(gt)), g.nbytes / 1e6))
print("H2D g pinned non_blocking %.3f ms" % tm(lambda: gdev.copy_(gpin, non_blocking=True)))
print("graph replay              %.3f ms" % tm(lambda: solver._execute(prog)))
uc = pool[lay["UC"]:lay["UC"] + nl * P, 0]
print("D2H UC .cpu()             %.3f ms  (%.1f MB)" % (tm(lambda: uc.cpu()), uc.numel() * 8 / 1e6))
ucpin = torch.empty(uc.shape, dtype=torch.float64, pin_memory=True)
print("D2H UC pinned             %.3f ms" % tm(lambda: ucpin.copy_(uc, non_blocking=True)))
print("D2H UC pinned + np.copy   %.3f ms" % tm(lambda: (ucpin.copy_(uc, non_blocking=True), torch.cuda.synchronize(), ucpin.numpy().copy())))
out = np.empty(uc.shape)
print("np.empty + copy_ into it  %.3f ms" % tm(lambda: torch.from_numpy(out).copy_(uc)))
uw = pool[:2 * N, 0]
print("D2H U|W .cpu()            %.3f ms  (%.1f MB)" % (tm(lambda: uw.cpu()), uw.numel() * 8 / 1e6))
print("_leaf_table(g) check      %.3f ms" % tm(lambda: solver._leaf_table(g)))

import cProfile
import pstats
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    solver.solve(f=f, g=gd)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
