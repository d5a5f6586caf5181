import sys, time
sys.path.insert(0, ".")
import torch
import bench
from paper_1612_02736_b200 import build_stage
from paper_1612_02736_b200.geometry import enumerate_gauss_nodes
for cfg in (5, 2):
    tree, spec, p, q, desc = bench.make_config(cfg, 0)
    plan = enumerate_gauss_nodes(tree, q)
    for rep in range(5):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        build_stage(tree, spec, p, q, plan=plan)
        torch.cuda.synchronize(); print(cfg, rep, round(time.perf_counter() - t0, 4), flush=True)
