"""cProfile of build_stage (host side) for a config: where the non-kernel time goes."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch

import bench
from paper_1612_02736_b200 import build_stage
from paper_1612_02736_b200.geometry import enumerate_gauss_nodes

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
tree, spec, p, q, desc = bench.make_config(cfg, 0)
plan = enumerate_gauss_nodes(tree, q)
build_stage(tree, spec, p, q, plan=plan)
torch.cuda.synchronize()
for _ in range(2):
    t0 = time.perf_counter()
    s = build_stage(tree, spec, p, q, plan=plan)
    torch.cuda.synchronize()
    print(f"build {time.perf_counter() - t0:.4f} s")
    del s
pr = cProfile.Profile()
pr.enable()
s = build_stage(tree, spec, p, q, plan=plan)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
