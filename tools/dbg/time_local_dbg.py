import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2405_12484_b200 import _abi, pdsolver, scenes
sc = scenes.make_scene("C3"); m = sc.mesh
ctx = _abi.Context(m.n_nodes, m.tets, m.shape_grad, m.volume, m.node_mass, sc.gammas.gamma_s, sc.gammas.gamma_v,
                   sc.pins, sc.dt, precision="fp32", tol=pdsolver.DEFAULT_TOL["fp32"])
ctx.set_state(m.nodes); ctx.set_pin_targets(sc.pin_targets); ctx.set_forces(sc.forces)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 60):
    ctx.step(30)
for reps in (1, 5, 20):
    print(reps, ctx.time_local(reps))
print("stats robust", ctx.stats()["robust"])
