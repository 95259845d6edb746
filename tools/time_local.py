"""k_local time per launch (event pair around each of 20 back-to-back launches) on a warmed C3 state;
the library is chosen by $VKPD_LIB (A/B of builds)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_12484_b200 import _abi, pdsolver, scenes  # noqa: E402
prec = sys.argv[1] if len(sys.argv) > 1 else "fp64"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 10
sc = scenes.make_scene("C3"); m = sc.mesh
ctx = _abi.Context(m.n_nodes, m.tets, m.shape_grad, m.volume, m.node_mass, sc.gammas.gamma_s, sc.gammas.gamma_v,
                   sc.pins, sc.dt, precision=prec, tol=pdsolver.DEFAULT_TOL[prec], nodes=m.nodes)
ctx.set_state(m.nodes); ctx.set_pin_targets(sc.pin_targets); ctx.set_forces(sc.forces)
for _ in range(frames):
    ctx.step(30)
kl, lp = ctx.time_local(20)
print(json.dumps({"lib": os.path.basename(os.environ.get("VKPD_LIB", "libvkpd.so")), "prec": prec, "frames": frames,
                  "k_local_ms": kl, "local_phase_ms": lp}))
