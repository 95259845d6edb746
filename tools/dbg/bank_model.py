"""Shared-memory bank model of k_cheb_reg's SpMV gathers (C3, float64).

Rebuilds the library's row layout on the host (patch_order: RCB patches, exported rows first;
build_cheb_neighbours: canonical entry order, halo slots) and counts, per warp and entry
position, the wavefronts of the 64-bit shared loads: a warp's LDS.64 is served per half-warp,
and a half-warp needs as many wavefronts as the most distinct slots that share a bank pair
(slot mod 16).  Compares orderings of the rows inside a patch, and bounds what re-assigning
entries to positions can reach (the bipartite edge colouring the library now does per warp in
vkpd.cu conflict_free_positions; the shipped image of d is 32-bit, served per 32-lane warp with
bank = slot mod 32, and the same colouring is applied with 32 lanes x 32 banks).

    python tools/dbg/bank_model.py [C3|C2]
"""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2405_12484_b200 import scenes  # noqa: E402

KOFF = 14


def rcb(X, ids, parts):
    nf = len(ids)
    chunk = -(-nf // parts)
    parts = -(-nf // chunk)
    out = list(ids)

    def split(lo, hi, p0, p1):
        if p1 - p0 <= 1 or hi - lo <= 1:
            out[lo:hi] = sorted(out[lo:hi])
            return
        seg = np.array(out[lo:hi])
        ext = X[seg].max(0) - X[seg].min(0)
        ax = int(np.argmax(ext))
        pm = (p0 + p1) // 2
        mid = min(hi, lo + (pm - p0) * chunk)
        order = np.lexsort((seg, X[seg, ax]))
        seg = seg[order]
        out[lo:hi] = list(seg)
        split(lo, mid, p0, pm)
        split(mid, hi, pm, p1)
    split(0, nf, 0, parts)
    return np.array(out), chunk


def adjacency(tets, n):
    a = np.concatenate([tets[:, [i, j]] for i in range(4) for j in range(4) if i != j])
    a = np.unique(a, axis=0)
    return a


def model(sc, reorder=None, parts=148):
    m = sc.mesh
    n = m.n_nodes
    pinned = np.zeros(n, bool); pinned[sc.pins] = True
    free = np.flatnonzero(~pinned)
    ids, chunk = rcb(m.nodes, free, parts)
    patch = -np.ones(n, int); patch[ids] = np.arange(len(ids)) // chunk
    e = adjacency(m.tets, n)
    pa, pb = patch[e[:, 0]], patch[e[:, 1]]
    expo = np.zeros(n, bool); expo[e[(pa >= 0) & (pb >= 0) & (pa != pb), 0]] = True
    nf = len(ids)
    for p in range(-(-nf // chunk)):
        lo, hi = p * chunk, min(nf, (p + 1) * chunk)
        seg = ids[lo:hi]
        if reorder is not None:
            seg = reorder(seg, m, expo)
        else:
            seg = np.concatenate([seg[expo[seg]], seg[~expo[seg]]])
        ids[lo:hi] = seg
    ioo = -np.ones(n, int); ioo[ids] = np.arange(nf)
    # rows' off-diagonal free columns, canonical order by caller-index offset
    fe = e[(ioo[e[:, 0]] >= 0) & (ioo[e[:, 1]] >= 0)]
    ri, ci = ioo[fe[:, 0]], ioo[fe[:, 1]]
    off = fe[:, 1] - fe[:, 0]
    order = np.lexsort((off, ri))
    ri, ci, off = ri[order], ci[order], off[order]
    start = np.searchsorted(ri, np.arange(nf))
    pos = np.arange(len(ri)) - start[ri]
    assert pos.max() < KOFF
    col = -np.ones((KOFF, nf), int)
    col[pos, ri] = ci
    threads = -(-chunk // 32) * 32
    wav = 0; req = 0
    for p in range(-(-nf // chunk)):
        r0, r1 = p * chunk, min(nf, (p + 1) * chunk)
        hslot = {}
        for o in range(KOFF):
            for i in range(r0, r1):
                c = col[o, i]
                if c >= 0 and not (r0 <= c < r1) and c not in hslot:
                    hslot[c] = None
        # grouped by owner (neighbour first-use order), then first use
        owners = []
        for c in hslot:
            ow = c // chunk
            if ow not in owners: owners.append(ow)
        hl = sorted(hslot, key=lambda c: owners.index(c // chunk))
        hs = {c: threads + j for j, c in enumerate(hl)}
        for o in range(KOFF):
            cs = col[o, r0:r1]
            loc = np.arange(r1 - r0)
            sl = np.where(cs < 0, loc, np.where((cs >= r0) & (cs < r1), cs - r0, 0))
            ext = (cs >= 0) & ((cs < r0) | (cs >= r1))
            sl[ext] = [hs[c] for c in cs[ext]]
            for w0 in range(0, r1 - r0, 32):
                req += 1
                for h0 in (w0, w0 + 16):
                    s = np.unique(sl[h0:min(h0 + 16, r1 - r0)])
                    if len(s) == 0:
                        continue
                    wav += np.bincount(s % 16, minlength=16).max()
    return wav / req


def by_grid(seg, m, expo):
    """Rows of a patch in grid order with the exported rows first (the current layout is the
    caller order, which for voxel meshes is this)."""
    return np.concatenate([seg[expo[seg]], seg[~expo[seg]]])


def coloring_bound(sc, parts=148):
    """Per half-warp lower bounds on wavefronts per position if entries are re-assigned to
    positions freely: max over bank classes of (edges) and of (distinct slots), vs 14."""
    import collections
    m = sc.mesh
    n = m.n_nodes
    pinned = np.zeros(n, bool); pinned[sc.pins] = True
    free = np.flatnonzero(~pinned)
    ids, chunk = rcb(m.nodes, free, parts)
    patch = -np.ones(n, int); patch[ids] = np.arange(len(ids)) // chunk
    e = adjacency(m.tets, n)
    pa, pb = patch[e[:, 0]], patch[e[:, 1]]
    expo = np.zeros(n, bool); expo[e[(pa >= 0) & (pb >= 0) & (pa != pb), 0]] = True
    nf = len(ids)
    for p in range(-(-nf // chunk)):
        lo, hi = p * chunk, min(nf, (p + 1) * chunk)
        seg = ids[lo:hi]
        ids[lo:hi] = np.concatenate([seg[expo[seg]], seg[~expo[seg]]])
    ioo = -np.ones(n, int); ioo[ids] = np.arange(nf)
    fe = e[(ioo[e[:, 0]] >= 0) & (ioo[e[:, 1]] >= 0)]
    ri, ci = ioo[fe[:, 0]], ioo[fe[:, 1]]
    rows = collections.defaultdict(list)
    for r, c in zip(ri, ci):
        rows[r].append(c)
    threads = -(-chunk // 32) * 32
    tot_e = tot_d = tot_cur = nh = 0
    for p in range(-(-nf // chunk)):
        r0, r1 = p * chunk, min(nf, (p + 1) * chunk)
        hs = {}
        for i in range(r0, r1):
            for c in rows[i]:
                if not (r0 <= c < r1) and c not in hs:
                    hs[c] = threads + len(hs)
        for h0 in range(r0, r1, 16):
            ce = np.zeros(16, int); slots = [set() for _ in range(16)]
            for i in range(h0, min(h0 + 16, r1)):
                for c in rows[i]:
                    s = c - r0 if r0 <= c < r1 else hs[c]
                    ce[s % 16] += 1; slots[s % 16].add(s)
            tot_e += max(14, ce.max()); tot_d += max(1, max(len(x) for x in slots)); nh += 1
    print("half-warps", nh, "mean max-class edges", tot_e / nh, "mean max-class distinct slots", tot_d / nh,
          "(ideal 14 wavefronts per half per plane over 14 positions)")


if __name__ == "__main__":
    key = sys.argv[1] if len(sys.argv) > 1 else "C3"
    sc = scenes.make_scene(key)
    print("nodes", sc.mesh.n_nodes, "caller order, exported first:", model(sc))
    print("caller order, no exported partition:", model(sc, reorder=lambda s, m, x: s))
    coloring_bound(sc)
