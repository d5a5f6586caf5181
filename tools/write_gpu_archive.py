"""Write reference-flavor archives from GPU-built solvers (stored + econ, refined mesh), plus the GPU
solves, into gpurun_out/; copied to tests/golden/ as fixtures for the reverse interop check
(tests/test_reference_objects.py: specdtn's own load_operators reads them)."""
import os
import sys

sys.path.insert(0, ".")
import numpy as np

from paper_1612_02736_b200 import RefinementSpec, build_stage, build_uniform_tree, catalog, refine_near_point
from paper_1612_02736_b200.archive import persist_operators

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
for mode in ("stored", "econ"):
    tree = build_uniform_tree((0.0, 1.0, 0.0, 1.0), 2)
    refine_near_point(tree, RefinementSpec((0.1, 0.1), 1))
    solver = build_stage(tree, catalog("manufactured", u="sin(pi*x1)*sin(pi*x2)"), 9, 8, mode)
    persist_operators(solver, os.path.join(out, f"gpu_archive_{mode}.sdtn"), flavor="reference")
    st = solver.solve(f=lambda pts: pts[:, 0] - 2 * pts[:, 1])
    ids = sorted(st.leaf_solutions)
    np.savez_compressed(os.path.join(out, f"gpu_archive_{mode}_solution.npz"), u=st.u, leaf_ids=np.array(ids),
                        leaf_sol=np.stack([st.leaf_solutions[i] for i in ids]))
print("ok")
