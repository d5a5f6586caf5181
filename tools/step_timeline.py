"""In-sequence (cold-L2) per-step timing of one solve: the sweep program run eagerly with CUDA
events between consecutive steps (host enqueues ahead of the GPU, so the GPU never idles)."""
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
solver = build_stage(tree, spec, p, q, plan=enumerate_gauss_nodes(tree, q))
prog = solver._program(args.nrhs)
lib = _ext.load()
s = torch.cuda.current_stream()
steps = [("up", st) for st in prog["up"]] + [("down", st) for st in prog["down"]]
for rep in range(4):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(steps) + 1)]
    torch.cuda.synchronize()
    ev[0].record()
    for i, (name, st) in enumerate(steps):
        lib.hps_sweep_gemv(st, s.cuda_stream)
        ev[i + 1].record()
    torch.cuda.synchronize()
tot = 0.0
for i, (name, st) in enumerate(steps):
    ms = ev[i].elapsed_time(ev[i + 1])
    tot += ms
    print(f"{name:4s} items={st.nitems:6d} R={st.R:5d} K={st.K:5d} mode2={st.mode2} {ms * 1e3:8.1f} us")
print(f"total {tot * 1e3:.1f} us (eager, events between steps)")
