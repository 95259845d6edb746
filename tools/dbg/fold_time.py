"""Device time of the C3 fold-window frame (frame-120 state of tests/golden/c3fold.npz): the
frame is re-run from the same state N times (graph), min / median ms and the robust count.
VKPD_LIB selects the library (A/B of builds)."""
import sys, os, json
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2405_12484_b200 import _abi, pdsolver, scenes  # noqa: E402
prec = sys.argv[1] if len(sys.argv) > 1 else "fp64"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
graph = (sys.argv[3] != "0") if len(sys.argv) > 3 else True
g = np.load("tests/golden/c3fold.npz")
sc = scenes.c3_sweater(); m = sc.mesh
ctx = _abi.Context(m.n_nodes, m.tets, m.shape_grad, m.volume, m.node_mass, sc.gammas.gamma_s, sc.gammas.gamma_v,
                   sc.pins, sc.dt, precision=prec, tol=pdsolver.DEFAULT_TOL[prec], nodes=m.nodes, use_graph=graph)
stream = torch.cuda.Stream()
ctx.set_stream(stream.cuda_stream)
ctx.set_pin_targets(sc.pin_targets); ctx.set_forces(sc.forces)
x0, v0 = g["x0"].astype(np.float64), g["v0"].astype(np.float64)
ms = []
for r in range(reps + 1):
    ctx.set_state(x0, v0)
    r0 = ctx.stats()["robust"]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream); ctx.step_async(30); e1.record(stream); ctx.sync()
    if r: ms.append(e0.elapsed_time(e1))
    rob = ctx.stats()["robust"] - r0
print(json.dumps({"lib": os.path.basename(os.environ.get("VKPD_LIB", "libvkpd.so")), "prec": prec,
                  "ms_min": min(ms), "ms_median": float(np.median(ms)), "robust": rob}))
