"""Where does simulate_mesh's end-to-end time go beyond the device frames? (C3, fp32)

Times 200 frames through pdsolver.simulate_mesh (fresh output array, as a user calls it) and
through the context's simulate() with a pre-faulted output array, to separate the cost of
first-touching the caller's frame stack from the copy pipeline itself.
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_12484_b200 import pdsolver, scenes  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
sc = scenes.c3_sweater()
m = sc.mesh
fseq = np.broadcast_to(sc.forces, (steps,) + sc.forces.shape).copy()
path = np.broadcast_to(sc.pin_targets, (steps,) + sc.pin_targets.shape).copy()
kw = dict(forces=fseq, pins=sc.pins, pin_targets=path, iterations=sc.iterations)
pdsolver.simulate_mesh(m, sc.gammas, 2, sc.dt, forces=fseq[:2], pins=sc.pins, pin_targets=path[:2],
                       iterations=sc.iterations)
res = {}
for rep in range(2):
    t0 = time.perf_counter()
    pdsolver.simulate_mesh(m, sc.gammas, steps, sc.dt, **kw)
    res[f"simulate_mesh_fresh_out_{rep}"] = (time.perf_counter() - t0) * 1e3 / steps
ctx = pdsolver.device_context(m, sc.gammas, sc.dt, sc.pins, "fp32", None, 0)
out = np.ones((steps, m.n_nodes, 3))
for rep in range(2):
    ctx.set_state(m.nodes, np.zeros_like(m.nodes))
    t0 = time.perf_counter()
    ctx.simulate(steps, sc.iterations, 1.0, forces=fseq, forces_per_step=True, pin_path=path, out=out)
    res[f"ctx_simulate_prefaulted_out_{rep}"] = (time.perf_counter() - t0) * 1e3 / steps
t0 = time.perf_counter()
a = np.empty((steps, m.n_nodes, 3))
a[...] = 1.0
res["first_touch_ms_per_frame_1thread"] = (time.perf_counter() - t0) * 1e3 / steps
print({k: round(v, 4) for k, v in res.items()})
