"""Domain-decomposed PD step across GPUs: one garment, one process per GPU.

Partition and exchange plan (host bookkeeping, deterministic, identical on every rank):
  * tets are labelled by slab (`partition_elements`, pdsolver.py:467-480) or by caller labels;
  * every node is owned by the lowest label among its incident tets;
  * rank r holds every tet touching a node it owns (its own tets plus a 1-ring of ghost
    tets), so the local step assembles complete residual rows for its owned nodes with no
    reduction; the non-owned nodes of those tets are its halo;
  * in rank r's device context the halo nodes are appended to the pinned list, so the
    local K_ff is exactly the owned-free block of the global K_ff and K_fp carries the
    coupling to the halo (pdsolver.py:210-229 applied per domain).

Per PD iteration (pdsolver.py:291-300) each rank runs the local step on its tets
(`vkpd_dev_residual`), then a distributed CG on the global K_ff: per iteration one halo
exchange of the search direction (point-to-point send/recv, NCCL over NVLink on GPUs),
one SpMV (`vkpd_dev_apply_K`) and two small all-reduces of per-column dot products.
After the solve the updated halo positions are exchanged once.  Vector algebra between
the library calls runs on torch tensors (the carrier).

`Comm` wraps torch.distributed: NCCL exchanges device tensors directly; the gloo
backend (CPU tests, or ranks sharing one GPU) stages through host memory.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .cms import partition_elements


@dataclass
class Part:
    rank: int
    owned: np.ndarray            # global ids of owned nodes (sorted)
    tets: np.ndarray             # global ids of local tets (sorted)
    nodes: np.ndarray            # global ids of local nodes (sorted)
    pins_owned: np.ndarray       # global ids of owned pinned nodes (global pin order)
    halo: np.ndarray             # global ids of halo nodes (sorted)
    local_tets: np.ndarray = None            # (nT, 4) local node ids
    send: dict = field(default_factory=dict)  # peer -> global ids this rank sends (sorted)
    recv: dict = field(default_factory=dict)  # peer -> global ids this rank receives (sorted)

    @property
    def ctx_pins_global(self):
        """Pinned list of the local context: owned pins (pin order) then halo."""
        return np.concatenate([self.pins_owned, self.halo]).astype(np.int64)


class DomainPlan:
    """Slab partition of a mesh into `n_parts` ranks with ghost tets and halo maps."""

    def __init__(self, mesh, pins, n_parts, labels=None):
        self.n_parts = int(n_parts)
        tets = np.asarray(mesh.tets, dtype=np.int64)
        nV, nE = mesh.n_nodes, len(tets)
        self.labels = partition_elements(mesh, n_parts, labels) if n_parts > 1 else np.zeros(nE, int)
        if self.labels.max() >= n_parts or self.labels.min() < 0:
            raise ValueError("labels must lie in [0, n_parts)")
        owner = np.full(nV, np.iinfo(np.int64).max, dtype=np.int64)
        np.minimum.at(owner, tets.reshape(-1), np.repeat(self.labels.astype(np.int64), 4))
        owner[owner == np.iinfo(np.int64).max] = 0          # isolated nodes
        self.owner = owner
        pins = np.asarray(pins, dtype=np.int64)
        self.pins = pins
        own_t = owner[tets]                                    # (nE, 4)
        self.parts = []
        for r in range(n_parts):
            owned = np.flatnonzero(owner == r)
            lt = np.flatnonzero((own_t == r).any(axis=1))
            nodes = np.union1d(np.unique(tets[lt]), owned)
            halo = np.setdiff1d(nodes, owned)
            pins_owned = pins[owner[pins] == r]
            part = Part(r, owned, lt, nodes, pins_owned, halo)
            part.local_tets = np.searchsorted(nodes, tets[lt])
            self.parts.append(part)
        for r, pr in enumerate(self.parts):
            for s, ps in enumerate(self.parts):
                if r == s:
                    continue
                common = np.intersect1d(pr.owned, ps.halo)
                if len(common):
                    pr.send[s] = common
                    ps.recv[r] = common

    def local_arrays(self, mesh, gammas, rank):
        """Local sub-mesh arrays of one rank (caller order = sorted global ids)."""
        p = self.parts[rank]
        return dict(n_nodes=len(p.nodes), tets=p.local_tets, shape_grad=mesh.shape_grad[p.tets],
                    volume=mesh.volume[p.tets], node_mass=mesh.node_mass[p.nodes],
                    gamma_s=np.asarray(gammas.gamma_s)[p.tets], gamma_v=np.asarray(gammas.gamma_v)[p.tets],
                    pins=np.searchsorted(p.nodes, p.ctx_pins_global))


class Comm:
    """Minimal collectives over torch.distributed (or a single rank)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.on = dist.is_available() and dist.is_initialized()
        self.group = group
        self.rank = dist.get_rank(group) if self.on else 0
        self.world = dist.get_world_size(group) if self.on else 1
        self.stage = self.on and dist.get_backend(group) == "gloo"

    def _to_wire(self, t):
        return t.cpu() if (self.stage and t.is_cuda) else t

    def allreduce_sum(self, t):
        if not self.on or self.world == 1:
            return t
        w = self._to_wire(t.contiguous())
        self.dist.all_reduce(w, op=self.dist.ReduceOp.SUM, group=self.group)
        return w.to(t.device) if w is not t else w

    def exchange(self, sends, recv_shapes, like):
        """sends: peer -> tensor; recv_shapes: peer -> shape; returns peer -> tensor."""
        if not self.on or self.world == 1 or (not sends and not recv_shapes):
            return {}
        import torch
        ops, out, wire = [], {}, {}
        for peer, shape in sorted(recv_shapes.items()):
            buf = torch.empty(shape, dtype=like.dtype, device="cpu" if self.stage else like.device)
            wire[peer] = buf
            ops.append(self.dist.P2POp(self.dist.irecv, buf, peer, group=self.group))
        for peer, t in sorted(sends.items()):
            ops.append(self.dist.P2POp(self.dist.isend, self._to_wire(t.contiguous()), peer, group=self.group))
        for req in self.dist.batch_isend_irecv(ops):
            req.wait()
        for peer, buf in wire.items():
            out[peer] = buf.to(like.device)
        return out


class CudaOps:
    """Local operators of one rank on its B200 (vkpd device-pointer primitives)."""

    def __init__(self, arrays, dt, precision="fp32", device=0):
        import torch
        from . import _abi
        self.torch = torch
        self.ctx = _abi.Context(arrays["n_nodes"], arrays["tets"], arrays["shape_grad"], arrays["volume"],
                                arrays["node_mass"], arrays["gamma_s"], arrays["gamma_v"], arrays["pins"], dt,
                                precision=precision, device=device, use_graph=False)
        self.dtype = torch.float32 if precision == "fp32" else torch.float64
        self.device = torch.device("cuda", device)
        stream = torch.cuda.current_stream(self.device)
        if stream.cuda_stream == 0:               # legacy default stream: give torch + library a real one
            stream = torch.cuda.Stream(self.device)
            torch.cuda.set_stream(stream)
        self.stream = stream
        self.ctx.set_stream(stream.cuda_stream)
        self.n, self.nF, self.nP, _ = self.ctx.sizes()
        self.int_of_orig = self.ctx.node_order()
        self.inv_diag = torch.empty(self.nF, dtype=self.dtype, device=self.device)
        if self.nF:
            self.ctx.dev_inv_diag(self.inv_diag.data_ptr())

    def residual(self, X, Xhat):
        R = self.torch.empty((self.nF, 4), dtype=self.dtype, device=self.device)
        if self.nF:
            self.ctx.dev_residual(X.data_ptr(), Xhat.data_ptr(), R.data_ptr())
        return R

    def apply_K(self, X):
        Y = self.torch.empty((self.nF, 4), dtype=self.dtype, device=self.device)
        if self.nF:
            self.ctx.dev_apply_K(X.data_ptr(), Y.data_ptr())
        return Y


class DistributedStepper:
    """One rank of the domain-decomposed PD step (`pd_step` semantics, no colliders)."""

    def __init__(self, plan, rank, mesh, gammas, dt, ops, comm, pin_targets=None, tol=2e-6, max_iters=1000):
        import torch
        self.torch = torch
        self.plan, self.rank, self.dt, self.ops, self.comm = plan, rank, float(dt), ops, comm
        self.tol, self.max_iters = float(tol), int(max_iters)
        p = plan.parts[rank]
        self.part = p
        ioo = ops.int_of_orig                                   # local -> internal
        self.ioo = torch.as_tensor(ioo, dtype=torch.long)
        self.nF, self.n = ops.nF, ops.n
        self.nPo = len(p.pins_owned)
        dev, dt_ = ops.device, ops.dtype
        self.dev, self.dtype = dev, dt_
        gl = p.nodes                                           # local -> global
        loc = {int(g): i for i, g in enumerate(gl)}
        def internal(gids):
            return torch.as_tensor(ioo[[loc[int(g)] for g in gids]], dtype=torch.long, device=dev)
        self.send_idx = {s: internal(g) for s, g in p.send.items()}
        self.recv_idx = {s: internal(g) for s, g in p.recv.items()}
        m = np.zeros(self.n)
        m[ioo] = mesh.node_mass[gl]
        self.m_dt2 = torch.as_tensor(m / self.dt ** 2, dtype=dt_, device=dev)
        inv_m = np.where(m > 0.0, 1.0 / np.where(m > 0.0, m, 1.0), 0.0)
        self.dt2_inv_m = torch.as_tensor(self.dt ** 2 * inv_m, dtype=dt_, device=dev)
        self.X = torch.zeros((self.n, 4), dtype=dt_, device=dev)
        self.V = torch.zeros_like(self.X)
        self.F = torch.zeros_like(self.X)
        self._pin_pos = {int(g): i for i, g in enumerate(plan.pins)}
        if pin_targets is None:
            self.set_pin_targets_local(np.zeros((self.nPo, 3)))
        else:
            self.set_pin_targets(pin_targets)

    # -- state in global numbering (full arrays; each rank uses its local nodes)
    def _to_internal(self, A):
        torch = self.torch
        out = torch.zeros((self.n, 4), dtype=self.dtype, device=self.dev)
        out[self.ioo.to(self.dev), :3] = torch.as_tensor(np.asarray(A)[self.part.nodes], dtype=self.dtype,
                                                         device=self.dev)
        return out

    def set_state(self, x, v=None):
        self.X = self._to_internal(x)
        self.V = self._to_internal(np.zeros_like(x) if v is None else v)

    def set_forces(self, f):
        self.F = self._to_internal(f) if f is not None else self.torch.zeros_like(self.X)

    def set_pin_targets_local(self, targets_owned):
        self.pin_tgt = self.torch.zeros((self.nPo, 4), dtype=self.dtype, device=self.dev)
        if self.nPo:
            self.pin_tgt[:, :3] = self.torch.as_tensor(np.asarray(targets_owned), dtype=self.dtype, device=self.dev)

    def set_pin_targets(self, targets_global_order):
        """targets for the global pin list (plan.pins order)."""
        idx = [self._pin_pos[int(g)] for g in self.part.pins_owned]
        self.set_pin_targets_local(np.asarray(targets_global_order, dtype=float).reshape(-1, 3)[idx]
                                   if self.nPo else np.zeros((0, 3)))

    def owned_positions(self):
        """(global ids, positions) of owned nodes."""
        X = self.X[:, :3].detach().cpu().numpy()
        ioo = self.ops.int_of_orig
        gl = self.part.nodes
        mask = np.isin(gl, self.part.owned)
        return gl[mask], X[ioo[mask]]

    # -- communication helpers
    def _halo(self, full):
        sends = {s: full[idx] for s, idx in self.send_idx.items()}
        shapes = {s: (len(idx), full.shape[1]) for s, idx in self.recv_idx.items()}
        got = self.comm.exchange(sends, shapes, full)
        for s, t in got.items():
            full[self.recv_idx[s]] = t
        return full

    def _allsum(self, t):
        return self.comm.allreduce_sum(t)

    # -- the step
    def step(self, iterations=30, damping=1.0, early_exit=True):
        """One PD step.  A round whose solve needs zero CG iterations leaves X unchanged, so
        every later round would repeat it exactly (same local step, same halo): with
        `early_exit` the loop stops there, as the single-GPU frame does.  The iteration count
        is identical on every rank (the residual norms are global)."""
        torch = self.torch
        nF, nPo = self.nF, self.nPo
        Xs, Vs = self.X.clone(), self.V.clone()
        Xhat = self.X + self.dt * self.V + self.dt2_inv_m[:, None] * self.F
        Xhat[:, 3] = 0
        X = Xhat.clone()
        if nPo:
            X[nF:nF + nPo] = self.pin_tgt
        X = self._halo(X)
        bb_loc = ((self.m_dt2[:nF, None] * Xhat[:nF, :3]).double() ** 2).sum()
        bb = float(self._allsum(bb_loc.reshape(1))[0])
        failed = -1
        for it in range(iterations):
            R = self.ops.residual(X, Xhat)
            Z = self.ops.inv_diag[:, None] * R
            P = torch.zeros_like(R)
            DX = torch.zeros_like(R)
            red = torch.cat([(R * Z).double().sum(0)[:3], (R * R).double().sum().reshape(1)])
            red = self._allsum(red)
            rz, rr = red[:3].clone(), float(red[3])
            rz_prev = torch.ones_like(rz)
            k = 0
            while rr > self.tol ** 2 * bb and k < self.max_iters:
                beta = torch.where((rz_prev != 0) & (k > 0), rz / torch.where(rz_prev != 0, rz_prev, 1.0),
                                   torch.zeros_like(rz))
                bvec = torch.cat([beta, beta.new_zeros(1)]).to(self.dtype)
                P = Z + bvec * P
                Pf = torch.zeros((self.n, 4), dtype=self.dtype, device=self.dev)
                Pf[:nF] = P
                Pf = self._halo(Pf)
                Q = self.ops.apply_K(Pf)
                pq = self._allsum((P * Q).double().sum(0)[:3])
                alpha = torch.where(pq != 0, rz / torch.where(pq != 0, pq, 1.0), torch.zeros_like(pq))
                avec = torch.cat([alpha, alpha.new_zeros(1)]).to(self.dtype)
                DX = DX + avec * P
                R = R - avec * Q
                Z = self.ops.inv_diag[:, None] * R
                red = self._allsum(torch.cat([(R * Z).double().sum(0)[:3], (R * R).double().sum().reshape(1)]))
                rz_prev, rz, rr = rz, red[:3].clone(), float(red[3])
                k += 1
            self.last_rounds = it + 1
            if k == 0 and early_exit:
                break
            X[:nF] = X[:nF] + DX
            X = self._halo(X)
            bad = torch.tensor([0.0 if bool(torch.isfinite(X[:nF]).all()) else 1.0], dtype=torch.float64,
                               device=self.dev)
            if float(self._allsum(bad)[0]) > 0 and failed < 0:
                failed = it
        if failed >= 0:
            self.X, self.V = Xs, Vs
            raise RuntimeError(f"projective step produced non-finite positions at iteration {failed}")
        self.V = damping * (X - Xs) / self.dt
        self.X = X
        return self
