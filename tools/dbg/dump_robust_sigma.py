"""Dump the sigma triples of the tets that take the robust SL(3) path at a given frame (dev probe input)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2405_12484_b200 import pdsolver, scenes
import oracle.pd_oracle as O

frame = int(sys.argv[1]); out = sys.argv[2]
sc = scenes.c3_sweater(); m = sc.mesh
fr = pdsolver.simulate_mesh(m, sc.gammas, frame, sc.dt, forces=sc.forces, pins=sc.pins,
                            pin_targets=sc.pin_targets, iterations=30, precision="fp32")
x = fr[-1]
F = O.deformation_gradients(x, m.tets, m.shape_grad)
U, sig, W = O.svd_rv(F)
s, lam, ok = O.kkt_newton_batch(sig)
feas = ok & (s.min(1) >= O.SV_FLOOR - 1e-12)
bounds = (sig.min(1) < 0.2) | (np.abs(sig).max(1) > 5.0)
sel = bounds | ~feas
if len(sys.argv) > 3 and sys.argv[3] == "all":
    sel = np.ones(len(sig), dtype=bool)
print("frame", frame, "bounds", int(bounds.sum()), "infeasible-first-start", int((~feas & ~bounds).sum()))
np.ascontiguousarray(sig[sel], dtype=np.float64).tofile(out)
q = sig[bounds]
print("sigma min quantiles", np.quantile(q.min(1), [0, .1, .5, .9, 1]) if len(q) else None)
print("sigma max quantiles", np.quantile(np.abs(q).max(1), [0, .1, .5, .9, 1]) if len(q) else None)
