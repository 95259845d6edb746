import ctypes as C, os, sys, collections
import numpy as np
sys.path.insert(0, os.getcwd())
os.environ["VKPD_LIB"] = "paper_2405_12484_b200/lib/libvkpd_trace.so"
from paper_2405_12484_b200 import _abi, pdsolver, scenes
sc = scenes.make_scene("C3"); m = sc.mesh
ctx = _abi.Context(m.n_nodes, m.tets, m.shape_grad, m.volume, m.node_mass, sc.gammas.gamma_s, sc.gammas.gamma_v,
                   sc.pins, sc.dt, precision="fp32", tol=1e-6)
ctx.set_state(m.nodes); ctx.set_pin_targets(sc.pin_targets); ctx.set_forces(sc.forces)
lib = _abi.load()
lib.vkpd_debug_pcg_trace.restype = C.c_int
buf = (C.c_ulonglong * 8192)()
for _ in range(10): ctx.step(30)
lib.vkpd_debug_pcg_trace(buf, 8192)
ctx.step(30)
n = lib.vkpd_debug_pcg_trace(buf, 8192)
ev = [(b >> 56, b & 0xffffffffffffff) for b in buf[:n]]
# segment into kernels by tag 0
kern = []; cur = None
for tag, t in ev:
    if tag == 0:
        cur = [(tag, t)]; kern.append(cur)
    elif cur is not None:
        cur.append((tag, t))
print("kernels", len(kern))
stats = collections.defaultdict(list)
for k in kern[:3]:
    print([ (tg, round((t - k[0][1]) / 1000, 2)) for tg, t in k][:40])
for k in kern:
    for (a, ta), (b, tb) in zip(k[:-1], k[1:]):
        stats[(a, b)].append((tb - ta) / 1000)
for key, v in sorted(stats.items()):
    print(key, "n", len(v), "mean us", round(np.mean(v), 3), "median", round(np.median(v), 3))
