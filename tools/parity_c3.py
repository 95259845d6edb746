"""Full-size parity evidence: C3 (390K tets) for a few frames, device fp32 and fp64 against the
CPU oracle (numpy/scipy restatement of the reference, pinned to its golden vectors).

    python tools/parity_c3.py --frames 3 --out profiles/r01b_parity_c3.json
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import pd_oracle as orc  # noqa: E402
from paper_2405_12484_b200 import pdsolver, scenes  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--frames", type=int, default=3)
p.add_argument("--out", default=None)
a = p.parse_args()
sc = scenes.c3_sweater()
m = sc.mesh
t0 = time.perf_counter()
ref = orc.simulate(m.nodes, m.tets, m.shape_grad, m.volume, sc.gammas.gamma_s, sc.gammas.gamma_v, m.node_mass,
                   a.frames, sc.dt, forces=sc.forces, pins=sc.pins, pin_targets=sc.pin_targets,
                   iterations=sc.iterations)
t_ref = time.perf_counter() - t0
out = {"workload": "C3-sweater-390K", "frames": a.frames, "oracle_s": round(t_ref, 1), "results": {}}
for prec in ("fp32", "fp64"):
    fr = pdsolver.simulate_mesh(m, sc.gammas, a.frames, sc.dt, forces=sc.forces, pins=sc.pins,
                                pin_targets=sc.pin_targets, iterations=sc.iterations, precision=prec)
    pos = [float(np.linalg.norm(fr[k] - ref[k]) / np.linalg.norm(ref[k])) for k in range(a.frames)]
    disp = [float(np.linalg.norm(fr[k] - ref[k]) / np.linalg.norm(ref[k] - m.nodes)) for k in range(a.frames)]
    out["results"][prec] = {"rel_l2_position": pos, "rel_l2_displacement": disp}
line = json.dumps(out)
print(line)
if a.out:
    open(a.out, "w").write(line + "\n")
