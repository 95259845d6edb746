"""Shared helpers for the test suite (not a test module)."""
import hashlib
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:32]


def scene_digest(sc):
    m = sc.mesh
    return digest(m.nodes, m.tets.astype(np.int64), m.node_mass, sc.gammas.gamma_s,
                  sc.gammas.gamma_v, sc.pins.astype(np.int64))


def rel_l2(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))
