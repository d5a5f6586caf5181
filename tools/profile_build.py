"""Phase timing of build_stage / solve on the GPU (CUDA events), for the perf loop."""
import argparse
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_1612_02736_b200 import build_stage, build_uniform_tree, problems, build_balanced_refined_tree
from paper_1612_02736_b200 import solver as S


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--n", type=int, default=0)
    args = ap.parse_args()
    cfg = args.config
    if cfg == 1:
        tree, spec, p, q = build_uniform_tree((0, 1, 0, 1), args.n or 4), problems.config1_spec(), 16, 15
    elif cfg == 2:
        tree, spec, p, q = build_uniform_tree((0, 1, 0, 1), args.n or 64), problems.config2_spec(), 16, 15
    elif cfg == 3:
        tree, spec, p, q = build_uniform_tree((0, 1, 0, 1), args.n or 32), problems.config3_spec(), 32, 31
    elif cfg == 4:
        tree, spec, p, q = build_balanced_refined_tree(8, (0.3, 0.7), 8), problems.config4_spec(), 16, 14
    else:
        tree, spec, p, q = build_uniform_tree((0, 1, 0, 1), args.n or 128), problems.config5_spec(1e-3), 16, 15
    from paper_1612_02736_b200.geometry import enumerate_gauss_nodes
    plan = enumerate_gauss_nodes(tree, q)
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        solver = build_stage(tree, spec, p, q, plan=plan, profile=(rep == 2))
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        print(f"cfg{cfg} build {t1 - t0:.4f} s (rep {rep})", flush=True)
    for name, ms in solver.phase_ms:
        print(f"   {ms:9.3f} ms  {name}")
    st = solver.solve()
    for rep in range(3):
        t0 = time.perf_counter()
        st = solver.solve()
        print(f"cfg{cfg} host solve {time.perf_counter() - t0:.4f} s", flush=True)
    lay = solver._layout
    nl = solver._n_leaves
    m = (p - 2) ** 2
    g = torch.zeros((nl * m, 1), dtype=torch.float64, device="cuda")
    f = torch.zeros((plan.node[tree.root].ext.size, 1), dtype=torch.float64, device="cuda")
    solver.solve_device(f, g)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        solver.solve_device(f, g)
    e1.record()
    torch.cuda.synchronize()
    print(f"cfg{cfg} device solve {e0.elapsed_time(e1) / 10:.3f} ms  retained {solver.device_bytes() / 1e9:.3f} GB", flush=True)


if __name__ == "__main__":
    main()
