"""Per-tet material container and the batched projections entry point.

`MaterialField` mirrors the reference container (`material.py:563-590`).
`batch_projections` is the drop-in for `material.batch_projections`
(`material.py:395-407`): it runs the sm_100a projection kernel through the
C-ABI library; there is no host fallback.
"""

from __future__ import annotations

import numpy as np

SV_FLOOR = 0.01          # material.py:25


class MaterialField:
    """Per-element coefficient pair (gamma_s, gamma_v), two flat float64 arrays."""

    def __init__(self, gamma_s, gamma_v):
        self.gamma_s = np.asarray(gamma_s, dtype=float)
        self.gamma_v = np.asarray(gamma_v, dtype=float)
        if self.gamma_s.shape != self.gamma_v.shape:
            raise ValueError("coefficient arrays must have matching shapes")

    @classmethod
    def uniform(cls, n_elements, gamma_s, gamma_v):
        return cls(np.full(n_elements, float(gamma_s)), np.full(n_elements, float(gamma_v)))

    def stacked(self):
        return np.concatenate([self.gamma_s, self.gamma_v])

    def copy(self):
        return MaterialField(self.gamma_s.copy(), self.gamma_v.copy())

    def __len__(self):
        return self.gamma_s.size


def batch_projections(F, precision="fp64"):
    """Rotation and volume projections (R, V) of a batch of F, on the GPU.

    F: (B, 3, 3) float.  Non-finite input raises ValueError like the reference.
    """
    from . import _abi
    F = np.ascontiguousarray(F, dtype=np.float64).reshape(-1, 3, 3)
    if not np.all(np.isfinite(F)):
        raise ValueError("non-finite deformation gradient in batch")
    return _abi.batch_projections(F, precision)


def projection_jacobians_batch(F):
    """Batched (d vec R / d vec F, d vec V / d vec F), each (B, 9, 9) (`material.py:490-524`).

    Row-major vec layout; float64 on the GPU (`vkpd_projection_jacobians`).
    """
    from . import _abi
    F = np.ascontiguousarray(F, dtype=np.float64).reshape(-1, 3, 3)
    if not np.all(np.isfinite(F)):
        raise ValueError("non-finite deformation gradient in batch")
    return _abi.projection_jacobians(F)
