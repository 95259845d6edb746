"""ctypes binding of the C-ABI library `lib/libvkpd.so` (declared in include/vkpd.h).

The library is the only compute path: if it is missing, or no CUDA device is
visible, every entry point raises -- there is no host fallback.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libvkpd.so")

VKPD_OK, VKPD_EINVAL, VKPD_ENONFINITE, VKPD_ECUDA = 0, 1, 2, 3
PRECISION = {"fp32": 32, "fp64": 64, 32: 32, 64: 64}

EXPORTS = (
    "vkpd_last_error", "vkpd_device_count", "vkpd_create", "vkpd_destroy", "vkpd_set_stream",
    "vkpd_get_stream", "vkpd_set_state", "vkpd_get_state", "vkpd_set_pin_targets",
    "vkpd_set_forces", "vkpd_step", "vkpd_step_async", "vkpd_sync", "vkpd_profile_step",
    "vkpd_elastic_rhs", "vkpd_global_solve", "vkpd_apply_K", "vkpd_get_stats",
    "vkpd_batch_projections", "vkpd_create_matrix", "vkpd_get_matrix_csr", "vkpd_a_jacobi_refine",
    "vkpd_power_rho", "vkpd_cms_set_basis", "vkpd_cms_solve", "vkpd_dev_residual", "vkpd_dev_apply_K",
    "vkpd_dev_inv_diag", "vkpd_get_node_order", "vkpd_get_sizes", "vkpd_set_colliders",
    "vkpd_set_gammas", "vkpd_set_yarn_interp", "vkpd_frame_outputs", "vkpd_v2y", "vkpd_equilibrium",
    "vkpd_projection_jacobians", "vkpd_hess_create", "vkpd_hess_destroy", "vkpd_hess_set_gammas",
    "vkpd_hess_energy_grad", "vkpd_hess_gamma_jt", "vkpd_hess_linearize", "vkpd_hess_csr",
    "vkpd_hess_apply", "vkpd_hess_solve", "vkpd_cms_set_blocks", "vkpd_cms_timing", "vkpd_time_local",
    "vkpd_step_cms", "vkpd_simulate", "vkpd_dev_cheb_step", "vkpd_get_gershgorin", "vkpd_set_state_dev",
    "vkpd_get_state_dev", "vkpd_set_forces_dev", "vkpd_set_pin_targets_dev", "vkpd_format_obj",
)


class MeshDesc(C.Structure):
    _fields_ = [
        ("n_nodes", C.c_int64), ("n_tets", C.c_int64), ("tets", C.c_void_p),
        ("shape_grad", C.c_void_p), ("volume", C.c_void_p), ("node_mass", C.c_void_p),
        ("gamma_s", C.c_void_p), ("gamma_v", C.c_void_p), ("pins", C.c_void_p),
        ("n_pins", C.c_int64), ("dt", C.c_double), ("nodes", C.c_void_p),
    ]


class Config(C.Structure):
    _fields_ = [
        ("precision", C.c_int), ("tol", C.c_double), ("max_iters", C.c_int), ("device", C.c_int),
        ("pcg_blocks", C.c_int), ("use_graph", C.c_int), ("solver", C.c_int),
        ("pd_early_exit", C.c_int), ("warm_rounds", C.c_int), ("unroll_rounds", C.c_int),
        ("tol_growth", C.c_double),
    ]


SOLVERS = {"auto": 0, "pcg": 1, "chebyshev": 2, "jacobi": 3}


class Stats(C.Structure):
    _fields_ = [
        ("n_pd_iters", C.c_int), ("cg_iters", C.c_int * 256), ("cg_iters_total", C.c_int),
        ("robust", C.c_uint), ("fallback", C.c_uint), ("pcg_blocks", C.c_int),
        ("ell_width", C.c_int), ("n_free", C.c_int64), ("local_ms", C.c_double * 256),
        ("global_ms", C.c_double * 256), ("pd_rounds_total", C.c_ulonglong), ("solver", C.c_int),
    ]


_lib = None


def load():
    """Load the shared library (once).  Raises ImportError when it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("VKPD_LIB", LIB_PATH)      # experiment builds live next to the default
    if not os.path.exists(path):
        raise ImportError(f"vkpd CUDA library not built: {path} (run __graft_entry__.build())")
    lib = C.CDLL(path)
    P = C.c_void_p
    I = C.c_int
    sig = {
        "vkpd_last_error": (C.c_char_p, []),
        "vkpd_device_count": (I, [C.POINTER(I)]),
        "vkpd_create": (I, [C.POINTER(MeshDesc), C.POINTER(Config), C.POINTER(P)]),
        "vkpd_destroy": (None, [P]),
        "vkpd_set_stream": (I, [P, P]),
        "vkpd_get_stream": (P, [P]),
        "vkpd_set_state": (I, [P, P, P]),
        "vkpd_get_state": (I, [P, P, P]),
        "vkpd_set_pin_targets": (I, [P, P]),
        "vkpd_set_forces": (I, [P, P]),
        "vkpd_step": (I, [P, I, C.c_double, C.POINTER(I)]),
        "vkpd_step_async": (I, [P, I, C.c_double]),
        "vkpd_sync": (I, [P, C.POINTER(I)]),
        "vkpd_profile_step": (I, [P, I, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                  C.POINTER(C.c_double)]),
        "vkpd_elastic_rhs": (I, [P, P, P, P, P, P]),
        "vkpd_global_solve": (I, [P, P, P, P, I]),
        "vkpd_apply_K": (I, [P, P, P]),
        "vkpd_get_stats": (I, [P, C.POINTER(Stats)]),
        "vkpd_batch_projections": (I, [I, C.c_int64, P, P, P, C.POINTER(C.c_uint), C.POINTER(C.c_uint)]),
        "vkpd_create_matrix": (I, [C.c_int64, P, P, P, P, C.c_int64, C.POINTER(Config), C.POINTER(P)]),
        "vkpd_get_matrix_csr": (I, [P, P, P, P, C.POINTER(C.c_int64)]),
        "vkpd_a_jacobi_refine": (I, [P, P, P, I, I, I, C.c_double, I, C.c_double, P, P, P, P]),
        "vkpd_power_rho": (I, [P, C.c_double, I, P, C.POINTER(C.c_double)]),
        "vkpd_cms_set_basis": (I, [P, I, P, P]),
        "vkpd_cms_solve": (I, [P, P, P, I, I, I, C.c_double, I, C.c_double, P]),
        "vkpd_dev_residual": (I, [P, P, P, P]),
        "vkpd_set_colliders": (I, [P, I, P, P, C.c_double]),
        "vkpd_dev_apply_K": (I, [P, P, P]),
        "vkpd_dev_inv_diag": (I, [P, P]),
        "vkpd_dev_cheb_step": (I, [P, P, P, P, P, C.c_double, C.c_double]),
        "vkpd_get_gershgorin": (I, [P, I, P]),
        "vkpd_set_state_dev": (I, [P, P, P]),
        "vkpd_get_state_dev": (I, [P, P, P]),
        "vkpd_set_forces_dev": (I, [P, P]),
        "vkpd_set_pin_targets_dev": (I, [P, P]),
        "vkpd_format_obj": (C.c_int64, [P, C.c_int64, P, C.c_int64, P, P, C.c_int64, C.c_char_p, P, C.c_int64]),
        "vkpd_get_node_order": (I, [P, P]),
        "vkpd_get_sizes": (I, [P, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                               C.POINTER(I)]),
        "vkpd_cms_set_blocks": (I, [P, I, P, P, P, P, P, I, C.c_int64, P, P]),
        "vkpd_cms_timing": (I, [P, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
        "vkpd_time_local": (I, [P, I, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
        "vkpd_step_cms": (I, [P, I, C.c_double, I, I, C.c_double, I, C.c_double, C.POINTER(I)]),
        "vkpd_simulate": (I, [P, I, I, C.c_double, P, I, P, P, C.POINTER(I), C.POINTER(I)]),
        "vkpd_hess_create": (I, [C.POINTER(MeshDesc), I, C.POINTER(P)]),
        "vkpd_hess_destroy": (None, [P]),
        "vkpd_hess_set_gammas": (I, [P, P, P]),
        "vkpd_hess_energy_grad": (I, [P, P, P, P]),
        "vkpd_hess_gamma_jt": (I, [P, P, P, P]),
        "vkpd_hess_linearize": (I, [P, P]),
        "vkpd_hess_csr": (I, [P, P, P, P, C.POINTER(C.c_int64)]),
        "vkpd_hess_apply": (I, [P, C.c_double, P, P]),
        "vkpd_hess_solve": (I, [P, C.c_double, C.c_double, P, P, C.c_double, I, C.POINTER(I),
                                C.POINTER(C.c_double)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class NonFiniteError(RuntimeError):
    pass


def check(rc):
    if rc == VKPD_OK:
        return
    msg = load().vkpd_last_error().decode(errors="replace")
    if rc == VKPD_EINVAL:
        raise ValueError(msg)
    if rc == VKPD_ENONFINITE:
        raise NonFiniteError(msg)
    raise RuntimeError(f"vkpd CUDA failure: {msg}")


def ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None:
        a = a.reshape(shape)
    return a


def device_count():
    n = C.c_int(0)
    load().vkpd_device_count(C.byref(n))
    return n.value


def batch_projections(F, precision="fp64"):
    lib = load()
    F = f64(F).reshape(-1, 3, 3)
    R = np.empty_like(F)
    V = np.empty_like(F)
    nr, nf = C.c_uint(0), C.c_uint(0)
    check(lib.vkpd_batch_projections(PRECISION[precision], F.shape[0], ptr(F), ptr(R), ptr(V),
                                     C.byref(nr), C.byref(nf)))
    if nf.value:
        import logging
        logging.getLogger("paper_2405_12484_b200.material").warning(
            "volume projection Newton failed for %d elements, using uniform scaling", nf.value)
    return R, V


class Context:
    """Owns one `vkpd_ctx` (device-resident scene)."""

    def __init__(self, nodes_count, tets, shape_grad, volume, node_mass, gamma_s, gamma_v, pins,
                 dt, precision="fp32", tol=0.0, max_iters=0, device=0, pcg_blocks=0, use_graph=True,
                 solver="auto", pd_early_exit=True, warm_rounds=-1, unroll_rounds=-1, nodes=None,
                 tol_growth=-1.0):
        self.lib = load()
        self._keep = dict(
            tets=np.ascontiguousarray(tets, dtype=np.int64).reshape(-1, 4),
            G=f64(shape_grad).reshape(-1, 4, 3),
            vol=f64(volume).reshape(-1),
            mass=None if node_mass is None else f64(node_mass).reshape(-1),
            gs=f64(gamma_s).reshape(-1),
            gv=f64(gamma_v).reshape(-1),
            pins=np.ascontiguousarray(pins, dtype=np.int64).reshape(-1),
            nodes=None if nodes is None else f64(nodes).reshape(-1, 3),
        )
        k = self._keep
        self.n = int(nodes_count)
        if k["nodes"] is not None and k["nodes"].shape[0] != self.n:
            raise ValueError("rest positions must be (n_nodes, 3)")
        self.n_tets = k["tets"].shape[0]
        self.n_pins = k["pins"].shape[0]
        if k["mass"] is None:
            raise ValueError("mesh node masses not lumped yet")
        d = MeshDesc(self.n, self.n_tets, ptr(k["tets"]), ptr(k["G"]), ptr(k["vol"]), ptr(k["mass"]),
                     ptr(k["gs"]), ptr(k["gv"]), ptr(k["pins"]) if self.n_pins else None,
                     self.n_pins, float(dt), ptr(k["nodes"]) if k["nodes"] is not None else None)
        if solver not in SOLVERS:
            raise ValueError(f"unknown solver {solver!r}")
        cfg = Config(PRECISION[precision], float(tol), int(max_iters), int(device), int(pcg_blocks),
                     1 if use_graph else 0, SOLVERS[solver], 1 if pd_early_exit else 0, int(warm_rounds),
                     int(unroll_rounds), float(tol_growth))
        h = C.c_void_p()
        check(self.lib.vkpd_create(C.byref(d), C.byref(cfg), C.byref(h)))
        self.h = h
        self.precision = precision
        self.dt = float(dt)

    def close(self):
        if getattr(self, "h", None):
            self.lib.vkpd_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:     # noqa: BLE001 - interpreter shutdown
            pass

    # -- state
    def set_stream(self, stream_ptr):
        check(self.lib.vkpd_set_stream(self.h, C.c_void_p(stream_ptr) if stream_ptr else None))

    def stream_ptr(self):
        return self.lib.vkpd_get_stream(self.h) or 0

    def set_state(self, x, v=None):
        x = f64(x, (self.n, 3))
        v = None if v is None else f64(v, (self.n, 3))
        check(self.lib.vkpd_set_state(self.h, ptr(x), ptr(v)))

    def get_state(self, want_x=True, want_v=True, out_x=None):
        x = (np.empty((self.n, 3)) if out_x is None else out_x) if want_x else None
        v = np.empty((self.n, 3)) if want_v else None
        check(self.lib.vkpd_get_state(self.h, ptr(x), ptr(v)))
        return x, v

    # -- state as torch CUDA tensors (the carrier): float64 (n, 3), caller order, no host copies
    def _dev(self, t, shape):
        if t is None:
            return None
        if not (getattr(t, "is_cuda", False)):
            raise TypeError("expected a CUDA tensor")
        import torch
        if t.dtype != torch.float64 or tuple(t.shape) != shape or not t.is_contiguous():
            raise ValueError(f"expected a contiguous float64 tensor of shape {shape}")
        return C.c_void_p(t.data_ptr())

    def set_state_tensor(self, x, v=None):
        check(self.lib.vkpd_set_state_dev(self.h, self._dev(x, (self.n, 3)), self._dev(v, (self.n, 3))))

    def get_state_tensor(self, x=None, v=None):
        """Positions / velocities into new (or given) float64 CUDA tensors, on the context stream."""
        import torch
        dev = torch.device("cuda", torch.cuda.current_device())
        x = torch.empty((self.n, 3), dtype=torch.float64, device=dev) if x is None else x
        v = torch.empty((self.n, 3), dtype=torch.float64, device=dev) if v is None else v
        check(self.lib.vkpd_get_state_dev(self.h, self._dev(x, (self.n, 3)), self._dev(v, (self.n, 3))))
        return x, v

    def set_forces_tensor(self, f):
        check(self.lib.vkpd_set_forces_dev(self.h, self._dev(f, (self.n, 3))))

    def set_pin_targets_tensor(self, t):
        if self.n_pins:
            check(self.lib.vkpd_set_pin_targets_dev(self.h, self._dev(t, (self.n_pins, 3))))

    def set_pin_targets(self, t):
        if self.n_pins:
            check(self.lib.vkpd_set_pin_targets(self.h, ptr(f64(t, (self.n_pins, 3)))))

    def set_forces(self, f):
        check(self.lib.vkpd_set_forces(self.h, None if f is None else ptr(f64(f, (self.n, 3)))))

    def set_yarn_interp(self, interp):
        """Yarn embedding interpolation matrix (n_yarn x n_nodes, CSR) for frame_outputs."""
        import scipy.sparse as sp
        A = sp.csr_matrix(interp)
        if A.shape[1] != self.n:
            raise ValueError("interpolation matrix has the wrong number of columns")
        ip = np.ascontiguousarray(A.indptr, dtype=np.int64)
        ix = np.ascontiguousarray(A.indices, dtype=np.int64)
        dv = np.ascontiguousarray(A.data, dtype=np.float64)
        check(self.lib.vkpd_set_yarn_interp(self.h, C.c_int64(A.shape[0]), ptr(ip), ptr(ix), ptr(dv)))
        self.n_yarn = A.shape[0]

    def frame_outputs(self, yarn=True, det=True):
        """(yarn positions interp @ x or None, max |det F - 1| or None) of the device state."""
        y = np.empty((getattr(self, "n_yarn", 0), 3)) if yarn else None
        d = C.c_double(0.0)
        check(self.lib.vkpd_frame_outputs(self.h, ptr(y), C.byref(d) if det else None))
        return y, (d.value if det else None)

    def equilibrium(self, inertia_target, x0, pin_vals, iterations):
        """pd_equilibrium rounds on the device (pdsolver.py:315-338); returns x (nV,3)."""
        a = f64(inertia_target, (self.n, 3))
        x0 = f64(x0, (self.n, 3))
        pv = f64(pin_vals, (self.n_pins, 3)) if self.n_pins else None
        out = np.empty((self.n, 3))
        failed = C.c_int(-1)
        check(self.lib.vkpd_equilibrium(self.h, ptr(a), ptr(x0), ptr(pv), int(iterations), ptr(out),
                                        C.byref(failed)))
        return out

    def set_gammas(self, gamma_s, gamma_v):
        """New per-tet material for the same mesh/pins/dt; K is re-assembled on the device."""
        ne = self.n_tets
        check(self.lib.vkpd_set_gammas(self.h, ptr(f64(gamma_s, (ne,))), ptr(f64(gamma_v, (ne,)))))

    def set_colliders(self, colliders, contact_stiffness=1e4):
        """colliders: sequence of ("plane", point, normal) / ("sphere", centre, radius)."""
        kinds, params = [], []
        for kind, *args in colliders:
            if kind == "plane":
                kinds.append(0)
                params.append(list(np.asarray(args[0], dtype=float)) + list(np.asarray(args[1], dtype=float)))
            elif kind == "sphere":
                kinds.append(1)
                params.append(list(np.asarray(args[0], dtype=float)) + [float(args[1]), 0.0, 0.0])
            else:
                raise ValueError(f"unknown collider kind {kind!r}")
        k = np.asarray(kinds, dtype=np.int32)
        p = np.asarray(params, dtype=np.float64).reshape(-1, 6)
        check(self.lib.vkpd_set_colliders(self.h, len(k), ptr(k) if len(k) else None, ptr(p) if len(k) else None,
                                          float(contact_stiffness)))

    def step(self, iterations, damping=1.0):
        fi = C.c_int(-1)
        rc = self.lib.vkpd_step(self.h, int(iterations), float(damping), C.byref(fi))
        check(rc)

    def step_async(self, iterations, damping=1.0):
        check(self.lib.vkpd_step_async(self.h, int(iterations), float(damping)))

    def sync(self):
        fi = C.c_int(-1)
        check(self.lib.vkpd_sync(self.h, C.byref(fi)))

    def simulate(self, steps, iterations, damping, forces=None, forces_per_step=False, pin_path=None, out=None):
        """`steps` frames from the current state (vkpd_simulate); returns (steps, nV, 3) float64."""
        frames = np.empty((steps, self.n, 3)) if out is None else out
        fo = None
        if forces is not None:
            # the reference indexes forces[i] / pin_path[i] (pdsolver.py:744-752): longer sequences
            # are fine, shorter ones raise as indexing would
            fo = f64(forces)
            if forces_per_step:
                fo = fo.reshape(-1, self.n, 3)
                if fo.shape[0] < steps:
                    raise IndexError(f"forces has {fo.shape[0]} steps, {steps} requested")
                fo = np.ascontiguousarray(fo[:steps])
            else:
                fo = fo.reshape(1, self.n, 3)
        pp = None
        if pin_path is not None and self.n_pins:
            pp = f64(pin_path).reshape(-1, self.n_pins, 3)
            if pp.shape[0] < steps:
                raise IndexError(f"pin path has {pp.shape[0]} steps, {steps} requested")
            pp = np.ascontiguousarray(pp[:steps])
        ff, fi = C.c_int(-1), C.c_int(-1)
        check(self.lib.vkpd_simulate(self.h, int(steps), int(iterations), float(damping), ptr(fo),
                                     1 if forces_per_step else 0, ptr(pp), ptr(frames), C.byref(ff), C.byref(fi)))
        return frames

    def step_cms(self, iterations, damping, sweeps, aggregation, omega, chebyshev, rho):
        """One pd_step with the cms global solver, entirely on the device."""
        fi = C.c_int(-1)
        check(self.lib.vkpd_step_cms(self.h, int(iterations), float(damping), int(sweeps), int(aggregation),
                                     float(omega), 1 if chebyshev else 0, float(rho), C.byref(fi)))

    def time_local(self, reps=20):
        """(k_local ms, local phase ms) per launch, back to back on the current state."""
        a, b = C.c_double(0.0), C.c_double(0.0)
        check(self.lib.vkpd_time_local(self.h, int(reps), C.byref(a), C.byref(b)))
        return a.value, b.value

    def profile_step(self, iterations, damping=1.0):
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        check(self.lib.vkpd_profile_step(self.h, int(iterations), float(damping), C.byref(a),
                                         C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    # -- parity entry points
    def elastic_rhs(self, x, with_frv=True):
        x = f64(x, (self.n, 3))
        rhs = np.empty((self.n, 3))
        F = R = V = None
        if with_frv:
            F, R, V = (np.empty((self.n_tets, 3, 3)) for _ in range(3))
        check(self.lib.vkpd_elastic_rhs(self.h, ptr(x), ptr(rhs), ptr(F), ptr(R), ptr(V)))
        return rhs, F, R, V

    def global_solve(self, B, pin_vals):
        B = f64(B)
        if B.ndim == 1:
            B = B[:, None]
        k = B.shape[1]
        P = f64(pin_vals).reshape(self.n_pins, k) if self.n_pins else np.zeros((0, k))
        X = np.empty_like(B)
        check(self.lib.vkpd_global_solve(self.h, ptr(B), ptr(P), ptr(X), int(k)))
        return X

    def apply_K(self, X):
        X = f64(X, (self.n, 3))
        Y = np.empty_like(X)
        check(self.lib.vkpd_apply_K(self.h, ptr(X), ptr(Y)))
        return Y

    def a_jacobi_refine(self, Bf, X0f, sweeps, aggregation, omega, chebyshev, rho):
        """Columns of Bf (n_free, k<=3) refined from X0f; returns (X, hist list per column, diverged)."""
        Bf = f64(Bf)
        X0f = f64(X0f)
        if Bf.ndim == 1:
            Bf, X0f = Bf[:, None], X0f[:, None]
        k = Bf.shape[1]
        steps = sweeps * aggregation if chebyshev else sweeps
        X = np.empty_like(Bf)
        hist = np.zeros((k, steps + 1))
        nh = np.zeros(k, dtype=np.int32)
        dv = np.zeros(k, dtype=np.int32)
        check(self.lib.vkpd_a_jacobi_refine(self.h, ptr(np.ascontiguousarray(Bf)), ptr(np.ascontiguousarray(X0f)),
                                            k, int(sweeps), int(aggregation), float(omega), int(bool(chebyshev)),
                                            float(rho), ptr(X), ptr(hist), ptr(nh), ptr(dv)))
        return X, [hist[c, :nh[c]].tolist() for c in range(k)], [bool(d) for d in dv]

    def power_rho(self, omega, v0, iters=30):
        rho = C.c_double(0.0)
        check(self.lib.vkpd_power_rho(self.h, float(omega), int(iters), ptr(f64(v0).reshape(-1)), C.byref(rho)))
        return rho.value

    def cms_set_basis(self, T, Kred_inv):
        T = np.asfortranarray(T, dtype=np.float64)
        Ki = np.asfortranarray(Kred_inv, dtype=np.float64)
        self._keep["cmsT"], self._keep["cmsKi"] = T, Ki
        check(self.lib.vkpd_cms_set_basis(self.h, T.shape[1], T.ctypes.data_as(C.c_void_p),
                                          Ki.ctypes.data_as(C.c_void_p)))

    def cms_set_blocks(self, blk):
        """Per-domain basis blocks (see cms.basis_blocks)."""
        i64 = lambda a: np.ascontiguousarray(a, dtype=np.int64)
        k = dict(rp=i64(blk["row_ptr"]), rows=i64(blk["rows"]), cp=i64(blk["col_ptr"]), cm=i64(blk["colmap"]),
                 A=f64(blk["A"]).reshape(-1), bnd=i64(blk["boundary"]), Ki=f64(blk["K_red_inv"]))
        self._keep["cms_blocks"] = k
        nd = len(k["rp"]) - 1
        check(self.lib.vkpd_cms_set_blocks(self.h, int(nd), ptr(k["rp"]), ptr(k["rows"]), ptr(k["cp"]), ptr(k["cm"]),
                                           ptr(k["A"]), int(blk["n_modes"]), C.c_int64(len(k["bnd"])),
                                           ptr(k["bnd"]), ptr(k["Ki"])))

    def cms_timing(self):
        a, b = C.c_double(0.0), C.c_double(0.0)
        check(self.lib.vkpd_cms_timing(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def cms_solve(self, B, pin_vals, sweeps, aggregation, omega, chebyshev, rho):
        B = f64(B)
        if B.ndim == 1:
            B = B[:, None]
        k = B.shape[1]
        P = f64(pin_vals).reshape(self.n_pins, k) if self.n_pins else np.zeros((0, k))
        X = np.empty_like(B)
        check(self.lib.vkpd_cms_solve(self.h, ptr(B), ptr(P), k, int(sweeps), int(aggregation), float(omega),
                                      int(bool(chebyshev)), float(rho), ptr(X)))
        return X

    # -- device-pointer primitives (torch tensors as carriers), dd.py
    def sizes(self):
        n, nf, npin, prec = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int()
        check(self.lib.vkpd_get_sizes(self.h, C.byref(n), C.byref(nf), C.byref(npin), C.byref(prec)))
        return n.value, nf.value, npin.value, prec.value

    def node_order(self):
        out = np.empty(self.n, dtype=np.int64)
        check(self.lib.vkpd_get_node_order(self.h, ptr(out)))
        return out

    def dev_residual(self, x_ptr, xhat_ptr, r_ptr):
        check(self.lib.vkpd_dev_residual(self.h, C.c_void_p(x_ptr), C.c_void_p(xhat_ptr), C.c_void_p(r_ptr)))

    def dev_apply_K(self, X_ptr, Y_ptr):
        check(self.lib.vkpd_dev_apply_K(self.h, C.c_void_p(X_ptr), C.c_void_p(Y_ptr)))

    def dev_inv_diag(self, out_ptr):
        check(self.lib.vkpd_dev_inv_diag(self.h, C.c_void_p(out_ptr)))

    def dev_cheb_step(self, d_ptr, res_ptr, y_ptr, dnext_ptr, c1, c2):
        check(self.lib.vkpd_dev_cheb_step(self.h, C.c_void_p(d_ptr), C.c_void_p(res_ptr), C.c_void_p(y_ptr),
                                          C.c_void_p(dnext_ptr), float(c1), float(c2)))

    def gershgorin(self, with_pinned_cols=False):
        g = C.c_double(0.0)
        check(self.lib.vkpd_get_gershgorin(self.h, 1 if with_pinned_cols else 0, C.byref(g)))
        return g.value

    def matrix_csr(self):
        nnz = C.c_int64(0)
        check(self.lib.vkpd_get_matrix_csr(self.h, None, None, None, C.byref(nnz)))
        indptr = np.empty(self.n + 1, dtype=np.int64)
        indices = np.empty(nnz.value, dtype=np.int64)
        data = np.empty(nnz.value)
        check(self.lib.vkpd_get_matrix_csr(self.h, ptr(indptr), ptr(indices), ptr(data), C.byref(nnz)))
        return indptr, indices, data

    def stats(self):
        st = Stats()
        check(self.lib.vkpd_get_stats(self.h, C.byref(st)))
        n = st.n_pd_iters
        return dict(cg_iters=list(st.cg_iters[:n]), cg_iters_total=st.cg_iters_total,
                    robust=st.robust, fallback=st.fallback, pcg_blocks=st.pcg_blocks,
                    ell_width=st.ell_width, n_free=st.n_free, local_ms=list(st.local_ms[:n]),
                    global_ms=list(st.global_ms[:n]), pd_rounds_total=st.pd_rounds_total,
                    solver={v: k for k, v in SOLVERS.items()}.get(st.solver, str(st.solver)))


def projection_jacobians(F):
    """(d vec R / d vec F, d vec V / d vec F), each (n, 9, 9), on the device."""
    F = f64(F).reshape(-1, 3, 3)
    n = F.shape[0]
    JR, JV = np.empty((n, 9, 9)), np.empty((n, 9, 9))
    check(load().vkpd_projection_jacobians(C.c_int64(n), ptr(F), ptr(JR), ptr(JV)))
    return JR, JV


def v2y(interp, x):
    """interp @ x on the device (float64, CSR order, no fused multiply-add)."""
    import scipy.sparse as sp
    A = sp.csr_matrix(interp)
    x = f64(x, (A.shape[1], 3))
    y = np.empty((A.shape[0], 3))
    ip = np.ascontiguousarray(A.indptr, dtype=np.int64)
    ix = np.ascontiguousarray(A.indices, dtype=np.int64)
    dv = np.ascontiguousarray(A.data, dtype=np.float64)
    check(load().vkpd_v2y(C.c_int64(A.shape[0]), ptr(ip), ptr(ix), ptr(dv), C.c_int64(A.shape[1]), ptr(x), ptr(y)))
    return y


class MatrixContext(Context):
    """Matrix-only device context: `GlobalSolver(K, free, pins)` (pdsolver.py:205-246)."""

    def __init__(self, K, pins, precision="fp64", tol=0.0, max_iters=0, device=0, pcg_blocks=0):
        import scipy.sparse as sp
        self.lib = load()
        K = sp.csr_matrix(K)
        K.sort_indices()
        self.n = K.shape[0]
        self.n_tets = 0
        pins = np.ascontiguousarray(pins, dtype=np.int64).reshape(-1)
        self.n_pins = len(pins)
        self._keep = dict(indptr=np.ascontiguousarray(K.indptr, dtype=np.int64),
                          indices=np.ascontiguousarray(K.indices, dtype=np.int64),
                          data=f64(K.data), pins=pins)
        k = self._keep
        cfg = Config(PRECISION[precision], float(tol), int(max_iters), int(device), int(pcg_blocks), 0,
                     SOLVERS["pcg"], 1, -1, -1, 1.0)
        h = C.c_void_p()
        check(self.lib.vkpd_create_matrix(self.n, ptr(k["indptr"]), ptr(k["indices"]), ptr(k["data"]),
                                          ptr(pins) if self.n_pins else None, self.n_pins,
                                          C.byref(cfg), C.byref(h)))
        self.h = h
        self.precision = precision


class HessContext:
    """Owns one `vkpd_hess` (float64 second-order machinery of one mesh, pin set and dt)."""

    def __init__(self, nodes_count, tets, shape_grad, volume, node_mass, gamma_s, gamma_v, pins, dt,
                 device=0):
        self.lib = load()
        self._keep = dict(
            tets=np.ascontiguousarray(tets, dtype=np.int64).reshape(-1, 4),
            G=f64(shape_grad).reshape(-1, 4, 3),
            vol=f64(volume).reshape(-1),
            mass=None if node_mass is None else f64(node_mass).reshape(-1),
            gs=f64(gamma_s).reshape(-1),
            gv=f64(gamma_v).reshape(-1),
            pins=np.ascontiguousarray(pins, dtype=np.int64).reshape(-1),
        )
        k = self._keep
        self.n = int(nodes_count)
        self.n_tets = k["tets"].shape[0]
        self.n_pins = k["pins"].shape[0]
        if k["mass"] is None:
            raise ValueError("mesh node masses not lumped yet")
        d = MeshDesc(self.n, self.n_tets, ptr(k["tets"]), ptr(k["G"]), ptr(k["vol"]), ptr(k["mass"]),
                     ptr(k["gs"]), ptr(k["gv"]), ptr(k["pins"]) if self.n_pins else None,
                     self.n_pins, float(dt))
        h = C.c_void_p()
        check(self.lib.vkpd_hess_create(C.byref(d), int(device), C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.lib.vkpd_hess_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_gammas(self, gamma_s, gamma_v):
        gs, gv = f64(gamma_s).reshape(-1), f64(gamma_v).reshape(-1)
        if gs.shape[0] != self.n_tets or gv.shape[0] != self.n_tets:
            raise ValueError("gamma arrays must have one entry per element")
        check(self.lib.vkpd_hess_set_gammas(self.h, ptr(gs), ptr(gv)))

    def energy_grad(self, x, want_energy=True, want_grad=True):
        x = f64(x, (self.n, 3))
        e = np.zeros(1)
        g = np.empty((self.n, 3)) if want_grad else None
        check(self.lib.vkpd_hess_energy_grad(self.h, ptr(x), ptr(e) if want_energy else None, ptr(g)))
        return (float(e[0]) if want_energy else None), g

    def gamma_jt(self, x, lam):
        x, lam = f64(x, (self.n, 3)), f64(lam, (self.n, 3))
        out = np.empty(2 * self.n_tets)
        check(self.lib.vkpd_hess_gamma_jt(self.h, ptr(x), ptr(lam), ptr(out)))
        return out

    def linearize(self, x):
        check(self.lib.vkpd_hess_linearize(self.h, ptr(f64(x, (self.n, 3)))))

    def csr(self):
        import scipy.sparse as sp
        nnz = C.c_int64(0)
        check(self.lib.vkpd_hess_csr(self.h, None, None, None, C.byref(nnz)))
        indptr = np.empty(3 * self.n + 1, dtype=np.int64)
        indices = np.empty(nnz.value, dtype=np.int64)
        data = np.empty(nnz.value)
        check(self.lib.vkpd_hess_csr(self.h, ptr(indptr), ptr(indices), ptr(data), C.byref(nnz)))
        return sp.csr_matrix((data, indices, indptr), shape=(3 * self.n, 3 * self.n))

    def apply(self, p, mass_scale=0.0):
        p = f64(p, (self.n, 3))
        y = np.empty((self.n, 3))
        check(self.lib.vkpd_hess_apply(self.h, float(mass_scale), ptr(p), ptr(y)))
        return y

    def solve(self, b, mass_scale=0.0, ridge=0.0, tol=1e-12, max_iters=0):
        """(H + s M/dt^2 + ridge I)_ff x_f = b_f; returns (x (nV,3), iterations, true relative residual)."""
        b = f64(b, (self.n, 3))
        x = np.empty((self.n, 3))
        it = C.c_int(0)
        rr = C.c_double(0.0)
        check(self.lib.vkpd_hess_solve(self.h, float(mass_scale), float(ridge), ptr(b), ptr(x), float(tol),
                                       int(max_iters), C.byref(it), C.byref(rr)))
        return x, it.value, rr.value
