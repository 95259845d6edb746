"""C2 100 frames in fp64 at several CG tolerances against the reference fixtures (margin study)."""
import os, sys, time, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2405_12484_b200 import pdsolver, scenes
g = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests/golden/c2.npz"))
sc = scenes.c2_scarf()
for tol in (1e-12, 3e-12, 1e-11):
    t = time.perf_counter()
    fr = pdsolver.simulate_mesh(sc.mesh, sc.gammas, 100, sc.dt, forces=sc.forces, pins=sc.pins,
                                pin_targets=sc.pin_targets, iterations=30, precision="fp64", tol=tol)
    dt = time.perf_counter() - t
    errs = {k: float(np.linalg.norm(fr[k-1] - g[f"frame{k}"]) / np.linalg.norm(g[f"frame{k}"])) for k in (1, 10, 100)}
    print(json.dumps({"tol": tol, "s": round(dt, 2), "rel_l2": errs}))
