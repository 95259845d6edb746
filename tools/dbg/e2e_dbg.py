import os, sys, time, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2405_12484_b200 import _abi, pdsolver, scenes
sc = scenes.make_scene("C3"); m = sc.mesh; steps = 200
fseq = np.broadcast_to(sc.forces, (steps,) + sc.forces.shape).copy()
path = np.broadcast_to(sc.pin_targets, (steps,) + sc.pin_targets.shape).copy()
pdsolver.simulate_mesh(m, sc.gammas, 2, sc.dt, forces=fseq[:2], pins=sc.pins, pin_targets=path[:2])
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    pdsolver.simulate_mesh(m, sc.gammas, steps, sc.dt, forces=fseq, pins=sc.pins, pin_targets=path)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print("simulate_mesh per-step forces+path ms/frame", 1e3 * (t1 - t0) / steps)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    pdsolver.simulate_mesh(m, sc.gammas, steps, sc.dt, forces=sc.forces, pins=sc.pins, pin_targets=sc.pin_targets)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print("simulate_mesh const forces ms/frame", 1e3 * (t1 - t0) / steps)
ctx = pdsolver.device_context(m, sc.gammas, sc.dt, sc.pins, "fp32")
ctx.set_state(m.nodes); ctx.set_pin_targets(sc.pin_targets); ctx.set_forces(sc.forces)
torch.cuda.synchronize(); t0 = time.perf_counter()
for k in range(steps):
    ctx.step_async(30)
ctx.sync(); t1 = time.perf_counter()
print("device-only async loop ms/frame (wall)", 1e3 * (t1 - t0) / steps)
