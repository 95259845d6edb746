"""Per-step phase timeline of the Chebyshev solver (block 0, globaltimer marks).
Build: nvcc ... -DVK_PCG_TRACE -shared -o paper_2405_12484_b200/lib/libvkpd_trace.so vkpd.cu"""
import ctypes as C, os, sys, collections, json
import numpy as np
sys.path.insert(0, os.getcwd())
os.environ.setdefault("VKPD_LIB", "paper_2405_12484_b200/lib/libvkpd_trace.so")
from paper_2405_12484_b200 import _abi, pdsolver, scenes
prec = sys.argv[1] if len(sys.argv) > 1 else "fp64"
sc = scenes.make_scene("C3"); m = sc.mesh
ctx = _abi.Context(m.n_nodes, m.tets, m.shape_grad, m.volume, m.node_mass, sc.gammas.gamma_s, sc.gammas.gamma_v,
                   sc.pins, sc.dt, precision=prec, tol=pdsolver.DEFAULT_TOL[prec], solver="chebyshev",
                   nodes=m.nodes)
ctx.set_state(m.nodes); ctx.set_pin_targets(sc.pin_targets); ctx.set_forces(sc.forces)
lib = _abi.load()
lib.vkpd_debug_pcg_trace.restype = C.c_int
buf = (C.c_ulonglong * 8192)()
for _ in range(6): ctx.step(30)
lib.vkpd_debug_pcg_trace(buf, 8192)
ctx.step(30)
n = lib.vkpd_debug_pcg_trace(buf, 8192)
ev = [(b >> 56, b & 0xffffffffffffff) for b in buf[:n]]
stats = collections.defaultdict(list)
for (a, ta), (b, tb) in zip(ev[:-1], ev[1:]):
    stats[(a, b)].append((tb - ta) / 1000)
for key, v in sorted(stats.items()):
    print(key, "n", len(v), "mean us", round(float(np.mean(v)), 3), "median", round(float(np.median(v)), 3))
