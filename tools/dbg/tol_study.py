import os, sys, json
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
from paper_2405_12484_b200 import _abi, pdsolver, scenes
from pdtest_helpers import golden, rel_l2
g3 = golden("c3.npz"); g2 = golden("c2.npz")
sc3 = scenes.c3_sweater(); sc2 = scenes.c2_scarf()
ref3 = sc3.mesh.nodes + g3["frame1"].astype(np.float64)
out = {}
for tol in (1e-6, 2e-6, 4e-6, 1e-5):
    pdsolver.invalidate_cache()
    fr = pdsolver.simulate_mesh(sc3.mesh, sc3.gammas, 1, sc3.dt, forces=sc3.forces, pins=sc3.pins,
                                pin_targets=sc3.pin_targets, iterations=30, precision="fp32", tol=tol)
    e3 = rel_l2(fr[0], ref3); d3 = rel_l2(fr[0] - sc3.mesh.nodes, g3["frame1"])
    fr2 = pdsolver.simulate_mesh(sc2.mesh, sc2.gammas, 100, sc2.dt, forces=sc2.forces, pins=sc2.pins,
                                 pin_targets=sc2.pin_targets, iterations=30, precision="fp32", tol=tol)
    e2 = [rel_l2(fr2[k - 1], g2[f"frame{k}"]) for k in (1, 10, 100)]
    ctx = pdsolver.device_context(sc3.mesh, sc3.gammas, sc3.dt, sc3.pins, "fp32", tol)
    out[tol] = {"c3_pos": e3, "c3_disp": d3, "c2_pos_1_10_100": e2, "c3_cg_last": ctx.stats()["cg_iters_total"]}
print(json.dumps(out, indent=1))
