"""Compare the backward-Euler stepper with and without the folded load (g = u_n/dt read in the
leaf steps' gathers) after a few steps; prints max differences per pool region."""
import os
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_1612_02736_b200 import build_stage, build_uniform_tree, problems
from paper_1612_02736_b200.timestepping import DeviceStepper, _leaf_points

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 4
dt = 1e-3
solver = build_stage(build_uniform_tree((0, 1, 0, 1), n), problems.config5_spec(dt), 16, 15)
pts = _leaf_points(solver).reshape(-1, 2)
u0 = torch.as_tensor(np.stack([problems.config5_initial(s)(pts).reshape(solver._n_leaves, -1) for s in range(nrhs)], -1),
                     device="cuda").contiguous()
bpts = solver.plan.coords[solver.plan.node[solver.tree.root].ext]
res = {}
for fold in ("0", "1"):
    os.environ["HPS_BE_FOLD"] = fold
    st = DeviceStepper(solver, nrhs, 1.0 / dt, 0.0)
    print("fold", fold, st.fold)
    st.set_state(u0)
    outs = []
    for k in range(1, 3):
        f = torch.as_tensor(np.repeat(problems.config5_dirichlet(bpts, k * dt)[:, None], nrhs, 1), device="cuda")
        st.step(f.contiguous())
        torch.cuda.synchronize()
        lay = st.lay
        N = solver.plan.n_gauss
        outs.append((st.pool[lay["U"]:lay["U"] + N].cpu().numpy().copy(), st.leaf_tabulations().cpu().numpy().copy(),
                     st.pool[lay["W"]:lay["W"] + N].cpu().numpy().copy()))
    res[fold] = outs
for k in range(2):
    for i, nm in enumerate(("U", "UC", "W")):
        a, b = res["0"][k][i], res["1"][k][i]
        print(k + 1, nm, np.abs(a - b).max(), np.abs(a).max())
