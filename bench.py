"""HPS build/solve benchmark (BASELINE.json metric) — one JSON line on rank 0.

Default workload = BASELINE.json configs[1] (config 2): variable-coefficient elliptic
problem on [0,1]^2, 64x64 leaves, p=16, q=15, N_cheb = 923,521, FP64.

  step   = one solve (upward + downward sweep, reference solver.py:337-354) of one batch of
           nrhs right-hand sides against the operators built once by build_stage
  value  = solve Mpts/s per RHS = N_cheb * nrhs / (seconds per step) / 1e6, whole job
           (summed over ranks), inputs resident in HBM
  e2e    = the same metric through the reference-facing API FactorizedSolver.solve(f, g)
           with host numpy inputs / outputs (H2D of f,g and D2H of u, w, h, leaf
           tabulations inside the timed region)
  build  = build_stage seconds, canonical FP64 TFLOP/s and fraction of the measured
           37.1 TFLOP/s DMMA peak (profiles/fp64_peaks_r01.jsonl)

--impl reference times the CPU oracle port (oracle/hps_oracle.py, a restatement of the
reference's numpy/scipy path) on the host cores with the same config/metric.
Multi-GPU (--gpus N under torchrun): independent replicas over disjoint RHS batches
(SURVEY.md 8e "data-parallel over RHS"), no data-path collective; timing max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAK_TFLOPS = 37.1     # measured DMMA m8n8k4 peak on this pool's B200 (tools/fp64_peaks.cu)
UNIT = (0.0, 1.0, 0.0, 1.0)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def make_config(cfg: int, n_override: int = 0):
    from paper_1612_02736_b200 import build_balanced_refined_tree, build_uniform_tree, problems
    if cfg == 1:
        return build_uniform_tree(UNIT, n_override or 4), problems.config1_spec(), 16, 15, "config1: Poisson 4x4 p=16"
    if cfg == 2:
        n = n_override or 64
        return (build_uniform_tree(UNIT, n), problems.config2_spec(), 16, 15,
                f"config2: var-coef elliptic {n}x{n} leaves p=16 q=15")
    if cfg == 3:
        n = n_override or 32
        return (build_uniform_tree(UNIT, n), problems.config3_spec(), 32, 31,
                f"config3: Helmholtz kappa=80 {n}x{n} leaves p=32 q=31")
    if cfg == 4:
        return (build_balanced_refined_tree(8, (0.3, 0.7), 8), problems.config4_spec(), 16, 14,
                "config4: 2:1-balanced refined quadtree (175 leaves) p=16 q=14")
    n = n_override or 128
    return (build_uniform_tree(UNIT, n), problems.config5_spec(1e-3), 16, 15,
            f"config5: backward-Euler heat {n}x{n} leaves p=16 q=15")


def canonical_build_flops(tree, plan, p, q):
    """leaf (2/3+4/3)m^3 + 2mcb + 2m^2b + 2bPb + 2bm^2; merge (2/3)m3^3 + 2m3^2 e + 2e^2 m3."""
    m, b, c, P = (p - 2) ** 2, 4 * q, 4 * (p - 1), p * p
    nleaf = sum(1 for n in tree.nodes if n.is_leaf)
    leaf = nleaf * (2.0 * m ** 3 + 2.0 * m * c * b + 2.0 * m * m * b + 2.0 * b * P * b + 2.0 * b * m * m)
    merge = 0.0
    for nid, node in enumerate(tree.nodes):
        if node.is_leaf:
            continue
        en = plan.node[nid]
        m3, e = en.j3.size, en.ext_mergeorder.size
        merge += (2.0 / 3.0) * m3 ** 3 + 2.0 * m3 * m3 * e + 2.0 * e * e * m3
        if en.wrap is not None:
            ec = en.ext.size
            merge += 2.0 * e * e * ec + 2.0 * ec * e * ec + 2.0 * m3 * e * ec
    return leaf, merge


def solve_bytes(tree, plan, p, q, nrhs):
    """Canonical retained-operator bytes + vector bytes per solve."""
    m, b, P = (p - 2) ** 2, 4 * q, p * p
    nleaf = sum(1 for n in tree.nodes if n.is_leaf)
    ops = nleaf * (m * b + m * m + b * m)
    vec = nleaf * (m + P) * nrhs
    for nid, node in enumerate(tree.nodes):
        if node.is_leaf:
            continue
        en = plan.node[nid]
        m3, e, ec = en.j3.size, en.ext_mergeorder.size, en.ext.size
        ops += m3 * m3 + m3 * ec + e * m3 + (2 * e * ec if en.wrap is not None else 0)
        vec += (2 * m3 + e + ec) * nrhs
    return 8.0 * ops, 8.0 * vec


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"hps_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.t_start = time.time()
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "50"], stdout=self.fh, stderr=subprocess.DEVNULL)
            # wait for the first sample so the timed region is covered from its start
            for _ in range(100):
                time.sleep(0.02)
                self.fh.flush()
                if os.path.getsize(self.path) > 0:
                    break
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()
            self.fh.close()

    def summary(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        with open(self.path) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 7:
                    rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for k, nm in enumerate(names):
                if r[3 + k].lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": float(rows[0][1]),
                "samples": len(rows), "reasons": sorted(reasons)}


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        backend = "nccl" if os.environ.get("HPS_BENCH_BACKEND", "nccl") == "nccl" else "gloo"
        if backend == "nccl":
            # one process per GPU: bind the device before the group so NCCL uses it
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group(backend)
    return rank, ws


def max_over_ranks(x, ws):
    if ws == 1:
        return x
    from paper_1612_02736_b200.replicas import max_over_ranks as _max
    return _max(x)


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        if dist.get_backend() == "nccl":
            dist.barrier(device_ids=[int(os.environ.get("LOCAL_RANK", "0"))])
        else:
            dist.barrier()


def config_dict(args, desc, nrhs, ncheb, ops_bytes, ws):
    """The `config` object, identical in both arms (the driver compares them)."""
    return {"workload": desc, "nrhs": nrhs, "N_cheb": ncheb,
            "l2": "operators (%.2f GB) exceed the 126 MB L2; no flush needed" % (ops_bytes / 1e9),
            "parallelism": f"replicas over RHS x{ws}" if ws > 1 else "1 GPU"}


def leaf_dict(tree, table_rows):
    """{leaf id: (m,) interior tabulation} in the reference's g convention (solver.py:241-253),
    built once outside any timed region; table_rows = rows of a (n_leaves, m) table in the
    solver's leaf-row order, paired with solver._leaf_ids."""
    ids, table = table_rows
    return {int(n): table[r] for r, n in enumerate(ids)}


# --------------------------------------------------------------------------- CPU reference arm

def cpu_solve_rate(tree, spec, p, q, plan, reps=1, threads=None):
    """Oracle (reference numpy/scipy restatement) build + timed solves; returns (Mpts/s per RHS, build s)."""
    from threadpoolctl import threadpool_limits
    from oracle import hps_oracle as orc
    from paper_1612_02736_b200.geometry import count_chebyshev_dofs
    ncheb = count_chebyshev_dofs(tree, p)
    with threadpool_limits(limits=threads):
        t0 = time.perf_counter()
        ops = orc.build(tree, spec, p, q, plan)
        tb = time.perf_counter() - t0
        root_ext = plan.node[tree.root].ext
        f = np.asarray(spec.dirichlet(plan.coords[root_ext]) if spec.dirichlet else np.zeros(root_ext.size))
        g = {}
        for lf in tree.leaves():
            geo = orc.leaf_geometry(p, q, lf.bounds.width, lf.bounds.height)
            pts = orc.leaf_points(lf.bounds, p, q)[geo["i_ci"]]
            g[lf.id] = spec.load(pts) if hasattr(spec, "load") else np.zeros(len(pts))
        orc.solve(ops, f, g)
        times = []
        for _ in range(reps):
            t0 = time.perf_counter()
            orc.solve(ops, f, g)
            times.append(time.perf_counter() - t0)
    ts = min(times)
    return ncheb / ts / 1e6, tb, ts


def best_threads(tree_small, spec, p, q):
    from paper_1612_02736_b200.geometry import enumerate_gauss_nodes
    plan = enumerate_gauss_nodes(tree_small, q)
    best, best_t = None, None
    for th in sorted({1, min(4, os.cpu_count() or 1), os.cpu_count() or 1}):
        _, tb, ts = cpu_solve_rate(tree_small, spec, p, q, plan, reps=1, threads=th)
        if best_t is None or tb + ts < best_t:
            best, best_t = th, tb + ts
    return best


def run_reference(args, rank, ws):
    if rank != 0:
        return
    from paper_1612_02736_b200.geometry import count_chebyshev_dofs, enumerate_gauss_nodes
    tree, spec, p, q, desc = make_config(args.config, args.n)
    small = make_config(args.config, 8 if args.config in (2, 5) else 4)[0] if args.config in (2, 3, 5) else tree
    th = best_threads(small, spec, p, q)
    plan = enumerate_gauss_nodes(tree, q)
    from threadpoolctl import threadpool_limits
    from oracle import hps_oracle as orc
    ncheb = count_chebyshev_dofs(tree, p)
    with threadpool_limits(limits=th):
        t0 = time.perf_counter()
        ops = orc.build(tree, spec, p, q, plan)
        build_s = time.perf_counter() - t0
        root_ext = plan.node[tree.root].ext
        f = np.asarray(spec.dirichlet(plan.coords[root_ext]) if spec.dirichlet else np.zeros(root_ext.size))
        g = {}
        for lf in tree.leaves():
            geo = orc.leaf_geometry(p, q, lf.bounds.width, lf.bounds.height)
            g[lf.id] = spec.load(orc.leaf_points(lf.bounds, p, q)[geo["i_ci"]])
        for _ in range(max(args.warmup, 1)):
            t1 = time.perf_counter()
            orc.solve(ops, f, g)
            t_one = time.perf_counter() - t1
        # bounded sample: at most ~90 s of timed CPU solves whatever K is
        timed = max(1, min(args.steps, int(90.0 / max(t_one, 1e-6))))
        t0 = time.perf_counter()
        for _ in range(timed):
            orc.solve(ops, f, g)
        el = time.perf_counter() - t0
    per = el / timed
    val = ncheb * args.nrhs / (per * args.nrhs) / 1e6
    lf, mf = canonical_build_flops(tree, plan, p, q)
    sb_ops, _ = solve_bytes(tree, plan, p, q, args.nrhs)
    line = {"impl": "reference", "metric": "HPS solve Mpts/s per RHS", "value": round(val, 4),
            "unit": "Mpts/s per RHS", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(per * 1e3, 3), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded manufactured solution, SURVEY.md 8d)",
            "config": config_dict(args, desc, args.nrhs, ncheb, sb_ops, ws),
            "cpu_baseline": {"value": round(val, 4), "unit": "Mpts/s per RHS", "cores": th,
                             "host_cores": os.cpu_count(), "kind": "port",
                             "sample": f"full workload; oracle/hps_oracle.py numpy/scipy, OPENBLAS threads={th} "
                                       f"(best of a 1/4/nproc sweep), {timed} timed solves (of K={args.steps}; "
                                       f"capped at ~90 s of CPU time)"},
            "e2e": {"value": round(val, 4), "unit": "Mpts/s per RHS", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "build": {"seconds": round(build_s, 3), "tflops": round((lf + mf) / build_s / 1e12, 5)}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU arm

def _node_depths(tree):
    depth = {tree.root: 0}
    stack = [tree.root]
    while stack:
        nid = stack.pop()
        for c in tree.nodes[nid].children:
            depth[c] = depth[nid] + 1
            stack.append(c)
    return depth


def _merge_flops(plan, nid):
    en = plan.node[nid]
    m3, e = en.j3.size, en.ext_mergeorder.size
    return (2.0 / 3.0) * m3 ** 3 + 2.0 * m3 * m3 * e + 2.0 * e * e * m3


def build_largest(reps=2):
    """North-star build target: FP64 tensor utilisation on the LARGEST batches,
    config 3's 1,024-leaf p=32 leaf stage (one hps_leaf_build) and config 5's top merge levels
    0-4 (31 merges, m3 up to 1,920). CUDA-event phase marks of build_stage(profile=True) around
    exactly those ABI calls; canonical FLOPs of SURVEY.md 8d; best of `reps` timed builds after
    one warm-up build."""
    import torch
    from paper_1612_02736_b200 import build_stage
    from paper_1612_02736_b200.geometry import enumerate_gauss_nodes
    out = {}
    for cfg in (3, 5):
        tree, spec, p, q, desc = make_config(cfg)
        plan = enumerate_gauss_nodes(tree, q)
        m, b, c, P = (p - 2) ** 2, 4 * q, 4 * (p - 1), p * p
        nleaf = sum(1 for n in tree.nodes if n.is_leaf)
        leaf_gf = nleaf * (2.0 * m ** 3 + 2.0 * m * c * b + 2.0 * m * m * b + 2.0 * b * P * b + 2.0 * b * m * m) / 1e9
        depth = _node_depths(tree)
        top = {d: sum(_merge_flops(plan, n) for n, dd in depth.items()
                      if dd == d and not tree.nodes[n].is_leaf) / 1e9 for d in range(5)}
        best = None
        for r in range(reps + 1):
            solver = build_stage(tree, spec, p, q, plan=plan, profile=True)
            ph = solver.phase_ms
            del solver
            torch.cuda.synchronize()
            leaf_ms = sum(ms for name, ms in ph if name.startswith("leaf-build"))
            merge_ms = {d: sum(ms for name, ms in ph if name.startswith(f"merge d{d} ")) for d in range(5)}
            if r == 0:
                continue  # warm-up
            if best is None or leaf_ms + sum(merge_ms.values()) < best[0] + sum(best[1].values()):
                best = (leaf_ms, merge_ms)
        leaf_ms, merge_ms = best
        if cfg == 3:
            out["config3_leaves"] = {
                "what": f"{nleaf} leaves p=32 (m=900) in one hps_leaf_build", "gflop": round(leaf_gf, 1),
                "ms": round(leaf_ms, 2), "tflops": round(leaf_gf / leaf_ms, 2),
                "frac_fp64_peak": round(leaf_gf / leaf_ms / FP64_PEAK_TFLOPS, 4)}
        else:
            gf = sum(top.values())
            ms = sum(merge_ms.values())
            out["config5_top_merges"] = {
                "what": "levels 0-4 (31 merges, m3 480-1920, e 1920-7680), hps_merge_build per level",
                "gflop": round(gf, 1), "ms": round(ms, 2), "tflops": round(gf / ms, 2),
                "frac_fp64_peak": round(gf / ms / FP64_PEAK_TFLOPS, 4),
                "per_level": {str(d): {"gflop": round(top[d], 1), "ms": round(merge_ms[d], 2),
                                       "frac_fp64_peak": round(top[d] / merge_ms[d] / FP64_PEAK_TFLOPS, 4)}
                              for d in range(5)}}
            out["config5_leaves"] = {
                "what": f"{nleaf} leaves p=16 (m=196) in one hps_leaf_build", "gflop": round(leaf_gf, 1),
                "ms": round(leaf_ms, 2), "tflops": round(leaf_gf / leaf_ms, 2),
                "frac_fp64_peak": round(leaf_gf / leaf_ms / FP64_PEAK_TFLOPS, 4)}
    out["fp64_peak_tflops"] = FP64_PEAK_TFLOPS
    out["peak_source"] = "measured DMMA m8n8k4 (tools/fp64_peaks.cu, profiles/fp64_peaks_r01.jsonl)"
    return out


def timestep_config5(hbm_peak, nts=20, nrhs=16):
    """North-star repeated workload: one backward-Euler step of config 5 (128x128 leaves, p=16,
    dt=1e-3) for 16 RHS through DeviceStepper: the graph-replayed 16-RHS solve whose leaf steps
    read g = u_n/dt from the device-resident leaf tabulations. Bytes = canonical solve bytes at
    nrhs=16 (operators once + vectors)."""
    import torch
    from paper_1612_02736_b200 import build_stage
    from paper_1612_02736_b200.geometry import count_chebyshev_dofs, enumerate_gauss_nodes
    from paper_1612_02736_b200.timestepping import DeviceStepper
    tree, spec, p, q, desc = make_config(5)
    plan = enumerate_gauss_nodes(tree, q)
    ncheb = count_chebyshev_dofs(tree, p)
    solver = build_stage(tree, spec, p, q, plan=plan)
    stp = DeviceStepper(solver, nrhs, 1.0 / float(spec.params["dt"]), 0.0)
    from paper_1612_02736_b200 import problems
    stp.set_state(torch.zeros_like(stp.leaf_tabulations()))
    bpts = plan.coords[plan.node[tree.root].ext]
    f16 = torch.as_tensor(np.repeat(problems.config5_dirichlet(bpts, 1e-3)[:, None], nrhs, axis=1),
                          device="cuda").contiguous()
    for _ in range(3):
        stp.step(f16)
    torch.cuda.synchronize()
    t0e, t1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0e.record()
    for _ in range(nts):
        stp.step(f16)
    t1e.record()
    torch.cuda.synchronize()
    tper = t0e.elapsed_time(t1e) / 1e3 / nts
    ops, vec = solve_bytes(tree, plan, p, q, nrhs)
    m = (p - 2) ** 2
    nleaf = solver._n_leaves
    # + the load formation g = u_n/dt (read m, write m per leaf per RHS) when it is a separate
    # launch; folded into the leaf steps' gathers (DeviceStepper.fold) it adds no traffic
    byts = ops + vec + (0.0 if stp.fold else 8.0 * nleaf * 2 * m * nrhs)
    fold = stp.fold
    del stp, solver
    return {"workload": desc, "nrhs": nrhs, "ms_per_step": round(tper * 1e3, 4),
            "Mpts_per_s_per_rhs": round(ncheb * nrhs / tper / 1e6, 1),
            "trajectory_1000_steps_s": round(tper * 1000, 3),
            "bytes_per_step": byts, "achieved_gbs": round(byts / tper / 1e9, 1),
            "frac_hbm": round(byts / tper / 1e9 / hbm_peak, 4),
            "what": ("graph-replayed 16-RHS solve with g = u_n/dt read from the leaf tabulations"
                     if fold else "hps_leaf_apply (g = u_n/dt) + graph-replayed 16-RHS solve")
                    + f", CUDA events, {nts} steps after 3 warm-up"}


def run_ours(args, rank, ws):
    import torch
    from paper_1612_02736_b200 import build_stage
    from paper_1612_02736_b200.geometry import count_chebyshev_dofs, enumerate_gauss_nodes
    from paper_1612_02736_b200 import _ext

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    hbm_peak, hbm_src = load_peaks()
    tree, spec, p, q, desc = make_config(args.config, args.n)
    plan = enumerate_gauss_nodes(tree, q)
    ncheb = count_chebyshev_dofs(tree, p)
    nrhs = args.nrhs
    m, P = (p - 2) ** 2, p * p

    # ---- build: timed after two warm-up builds (the first calls pay lazy CUDA/module init and the
    # device / pinned-host caching allocators' first cudaMalloc / cudaHostAlloc); the cold first
    # build is reported alongside
    t0 = time.perf_counter()
    build_stage(tree, spec, p, q, plan=plan)
    torch.cuda.synchronize()
    build_cold = time.perf_counter() - t0
    build_stage(tree, spec, p, q, plan=plan)
    torch.cuda.synchronize()
    barrier(ws)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    solver = build_stage(tree, spec, p, q, plan=plan)
    e1.record()
    torch.cuda.synchronize()
    build_wall = time.perf_counter() - t0
    build_dev = e0.elapsed_time(e1) / 1e3
    lf, mf = canonical_build_flops(tree, plan, p, q)
    build_s = max_over_ranks(build_wall, ws)

    # ---- device-resident inputs (seeded): f on the root boundary, g interior loads
    rng = np.random.default_rng(1234 + rank)
    root_ext = plan.node[tree.root].ext
    f_host = np.asarray(spec.dirichlet(plan.coords[root_ext]) if spec.dirichlet else np.zeros(root_ext.size))
    g_host = solver._leaf_table(None)
    f_dev = torch.as_tensor(np.repeat(f_host[:, None], nrhs, axis=1) * (1.0 + 0.01 * rng.standard_normal(nrhs)),
                            device="cuda").contiguous()
    g_dev = torch.as_tensor(np.repeat(g_host.reshape(-1, 1), nrhs, axis=1), device="cuda").contiguous()
    prog = solver._program(nrhs)
    launches_per_step = len(prog["up"]) + len(prog["down"]) + 1  # + the Dirichlet copy

    for _ in range(args.warmup):
        solver.solve_device(f_dev, g_dev)
    torch.cuda.synchronize()
    barrier(ws)
    with ClockSampler(local) as clk:
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(args.steps):
            solver.solve_device(f_dev, g_dev)
        ev1.record()
        torch.cuda.synchronize()
        el = ev0.elapsed_time(ev1) / 1e3
    el = max_over_ranks(el, ws)
    per = el / args.steps
    value = ncheb * nrhs * ws / per / 1e6

    # ---- dominant kernel: leaf downward sweep ([F|S] [g; u_ext]), timed alone on the stream
    lib = _ext.load()
    sptr = torch.cuda.current_stream().cuda_stream
    ngrp = len(solver.leaf_groups)
    leaf_down = list(prog["down"][-ngrp:])
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    k0.record()
    for _ in range(reps):
        for st in leaf_down:
            lib.hps_sweep_gemv(st, sptr)
    k1.record()
    torch.cuda.synchronize()
    kt = k0.elapsed_time(k1) / 1e3 / reps
    nleaf = solver._n_leaves
    b = 4 * q
    c_ext = 4 * (p - 1)
    kbytes = 8.0 * nleaf * (m * (m + b) + (m + b) * nrhs + (m + c_ext) * nrhs)
    achieved = kbytes / kt / 1e9

    # ---- e2e through the public host API in the reference's own input convention: f as an
    # array on the root exterior, g as a {leaf id: (m,)} mapping; host numpy in,
    # host numpy out (SolveState.u, w, h_root, every leaf tabulation)
    g_tab = solver._leaf_table(None)
    g_dict = leaf_dict(tree, (solver._leaf_ids, g_tab))
    e2e_steps = max(1, min(args.steps, 20))
    for _ in range(max(args.warmup, 3)):
        st = solver.solve(f=f_host, g=g_dict)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        st = solver.solve(f=f_host, g=g_dict)
    e2e_t = (time.perf_counter() - t0) / e2e_steps
    e2e_t = max_over_ranks(e2e_t, ws)
    del st
    lay = solver._layout
    h2d = 8 * (root_ext.size + g_tab.size)
    # read back: u | w (2 N_gauss), h_root and the leaf tabulations (n_leaves x p^2)
    d2h = 8 * (2 * solver.plan.n_gauss + lay["hsize"][tree.root] + solver._n_leaves * p * p)

    # ---- CPU baseline: oracle on a bounded sample (rank 0, N=1 only)
    cpu = None
    if rank == 0 and ws == 1 and not args.skip_cpu:
        n_s = {1: 4, 2: 16, 3: 8, 4: 0, 5: 16}[args.config]
        stree, sspec, _, _, sdesc = make_config(args.config, n_s) if n_s else (tree, spec, p, q, desc)
        splan = enumerate_gauss_nodes(stree, q)
        th = min(4, os.cpu_count() or 1)
        rate, tb, ts = cpu_solve_rate(stree, sspec, p, q, splan, reps=3, threads=th)
        cpu = {"value": round(rate, 4), "unit": "Mpts/s per RHS", "cores": th, "host_cores": os.cpu_count(),
               "kind": "port",
               "sample": f"{sdesc}: oracle build ({tb:.1f} s) + best of 3 solves ({ts * 1e3:.1f} ms), "
                         f"OPENBLAS threads={th}"}

    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            tr = json.load(fh).get(f"config{args.config}:leaf_down_gemv_nrhs{nrhs}")
        if tr and args.n in (0, 64):
            traffic = tr["dram_bytes_read"] + tr["dram_bytes_write"]
    except Exception:
        traffic = None
    sb_ops, sb_vec = solve_bytes(tree, plan, p, q, nrhs)
    line = {
        "metric": "HPS solve Mpts/s per RHS", "value": round(value, 3), "unit": "Mpts/s per RHS",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(per * 1e3, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded manufactured solution / loads, SURVEY.md 8d; no dataset)",
        "config": config_dict(args, desc, nrhs, ncheb, sb_ops, ws),
        "roofline": {"bound": "hbm", "kernel": "sweep_kernel (leaf downward sweep, [F|S][g;u_ge] + L u_ge)", "achieved": round(achieved, 1),
                     "peak": hbm_peak, "unit": "GB/s", "frac": round(achieved / hbm_peak, 4), "traffic": traffic,
                     "algorithmic_bytes": kbytes,
                     "peak_source": hbm_src,
                     # the copy peak counts read+write bytes; a read-only stream can exceed it
                     "frac_of_datasheet_7700": round(achieved / 7700.0, 4)},
        "solve_roofline": {"bytes_per_step": sb_ops + sb_vec, "achieved_gbs": round((sb_ops + sb_vec) / per / 1e9, 1),
                           "frac": round((sb_ops + sb_vec) / per / 1e9 / hbm_peak, 4)},
        "build": {"seconds": round(build_s, 4), "device_seconds": round(build_dev, 4),
                  "cold_first_call_seconds": round(build_cold, 4),
                  "gflop_canonical": round((lf + mf) / 1e9, 2),
                  "tflops": round((lf + mf) / build_dev / 1e12, 3),
                  "frac_fp64_peak": round((lf + mf) / build_dev / 1e12 / FP64_PEAK_TFLOPS, 4),
                  "fp64_peak_tflops": FP64_PEAK_TFLOPS,
                  # Y = T_ei X per parent (solve-time operator, built on the first solve)
                  "solve_prep_seconds": round(getattr(solver, "prep_seconds", 0.0), 4)},
        "e2e": {"value": round(ncheb * ws / e2e_t / 1e6, 3), "unit": "Mpts/s per RHS", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "cpu_baseline": cpu,
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk.summary(),
    }
    if not args.no_extras and rank == 0:
        # north-star targets beyond the headline metric, in their own
        # clock-sampled region after the timed solve loop
        del solver, prog
        torch.cuda.empty_cache()
        with ClockSampler(local) as clk2:
            extra = {"build_largest": build_largest(), "timestep": timestep_config5(hbm_peak)}
        extra["clocks"] = clk2.summary()
        line["north_star"] = extra
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--nrhs", type=int, default=1)
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the north-star build/timestep measurements (config 3 and 5 builds)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    rank, ws = dist_init()
    if args.impl == "reference":
        run_reference(args, rank, ws)
    else:
        run_ours(args, rank, ws)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
