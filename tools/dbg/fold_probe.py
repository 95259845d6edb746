import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from paper_2405_12484_b200 import _abi, pdsolver, scenes
g = np.load('tests/golden/c3fold.npz')
sc = scenes.c3_sweater(); m = sc.mesh
def rel(a, b): return float(np.linalg.norm(a - b) / np.linalg.norm(b))
for prec in ("fp64", "fp32"):
    x0, v0 = g["x0"].astype(np.float64), g["v0"].astype(np.float64)
    ctx = _abi.Context(m.n_nodes, m.tets, m.shape_grad, m.volume, m.node_mass, sc.gammas.gamma_s, sc.gammas.gamma_v,
                       sc.pins, sc.dt, precision=prec, tol=pdsolver.DEFAULT_TOL[prec], nodes=m.nodes)
    ctx.set_state(x0, v0); ctx.set_pin_targets(sc.pin_targets); ctx.set_forces(sc.forces)
    r0 = ctx.stats()["robust"]; ctx.step(30); x, v = ctx.get_state()
    print(prec, "robust", ctx.stats()["robust"] - r0, "pos", rel(x, x0 + g["disp"]), "disp", rel(x - x0, g["disp"]), "v", rel(v, g["v"]))
