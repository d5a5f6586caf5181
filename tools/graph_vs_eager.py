"""Whole-solve time: CUDA-graph replay vs eager launches of the same sweep program."""
import sys
sys.path.insert(0, ".")
import torch
import bench
from paper_1612_02736_b200 import build_stage
from paper_1612_02736_b200.geometry import enumerate_gauss_nodes

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 16
tree, spec, p, q, desc = bench.make_config(cfg, 0)
solver = build_stage(tree, spec, p, q, plan=enumerate_gauss_nodes(tree, q))
prog = solver._program(nrhs)
for mode in (True, False, True):
    solver.use_graphs = mode
    for _ in range(3):
        solver._execute(prog)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        solver._execute(prog)
    e1.record()
    torch.cuda.synchronize()
    print(f"cfg{cfg} nrhs={nrhs} graphs={mode}: {e0.elapsed_time(e1) / 20:.4f} ms per solve "
          f"({len(prog['up']) + len(prog['down']) + 1} launches)")
