"""Mesh-to-yarn transfer of the per-frame output step.

`v2y` mirrors `transfer.v2y` (`transfer.py:26-28` of the reference): yarn vertex
positions are the embedding's barycentric interpolation of the mesh nodes.  The
product runs on the device (`vkpd_v2y`), in CSR order with separately rounded
multiply and add, so it returns the same float64 bits as the reference's
`embedding.interp @ x`.  Inside a simulation the same product runs on the
device-resident state: `Context.set_yarn_interp` + `Context.frame_outputs`, which
also returns the det(F) deviation the reference's simulate loop records
(`cli.py:639-640`).
"""

from __future__ import annotations

from . import _abi


def v2y(embedding, node_positions):
    """Yarn vertex positions interpolated from mesh node positions.

    `embedding` is a reference `YarnEmbedding` (its `.interp`) or the
    interpolation matrix itself.
    """
    interp = getattr(embedding, "interp", embedding)
    return _abi.v2y(interp, node_positions)
