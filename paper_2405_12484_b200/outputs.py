"""Per-frame outputs of `volknit simulate`: OBJ frames, `timings.csv`,
`sim_report.json` (`cli.py:538-547, 596-656`).

The reference's `cmd_simulate` steps the garment frame by frame and, after each step, computes
the worst |det F - 1| over the tets (`cli.py:639-640`), transfers the volume positions to the yarn
vertices (`transfer.v2y`), and writes `frames/mesh_NNNN.obj` (the enclosure's boundary
triangles) and `frames/yarn_NNNN.obj` (the yarn polylines); at the end it writes `timings.csv`
(stage, milliseconds) and `sim_report.json`.  Here the step, the det deviation and the yarn
transfer run on the device (`vkpd_frame_outputs`), the OBJ text is formatted by the library's
host formatter (`vkpd_format_obj`, %.17g like Python's ".17g": byte-identical files), and a
writer thread puts frame k on disk while frame k+1 computes.  The yarn-model sequence files
(`yarn_model.write_sequence`) belong to the yarn model, which SURVEY.md 2 keeps out of scope;
the yarn positions per frame are returned to the caller.
"""

from __future__ import annotations

import ctypes as C
import json
import os
import queue
import threading
import time

import numpy as np

from . import _abi

__all__ = ["format_obj", "write_obj", "write_csv", "write_report", "simulate_to_disk"]


def _fmt(v):
    if isinstance(v, (float, np.floating)):
        return f"{float(v):.17g}"
    return str(v)


def format_obj(vertices, faces=None, lines=None, comment=None):
    """OBJ text (bytes) of `_write_obj` (`cli.py:538-547`), formatted in the library."""
    lib = _abi.load()
    v = np.ascontiguousarray(vertices, dtype=np.float64).reshape(-1, 3)
    f = None if faces is None else np.ascontiguousarray(faces, dtype=np.int64).reshape(-1, 3)
    lp = li = None
    nl = 0
    if lines is not None:
        runs = [np.asarray(r, dtype=np.int64).reshape(-1) for r in lines]
        nl = len(runs)
        lp = np.zeros(nl + 1, dtype=np.int64)
        lp[1:] = np.cumsum([len(r) for r in runs])
        li = np.concatenate(runs) if runs else np.zeros(0, dtype=np.int64)
    cm = comment.encode() if comment else None
    args = (_abi.ptr(v), len(v), _abi.ptr(f) if f is not None else None, 0 if f is None else len(f),
            _abi.ptr(lp) if lp is not None else None, _abi.ptr(li) if li is not None and len(li) else None, nl, cm)
    n = lib.vkpd_format_obj(*args, None, 0)
    buf = C.create_string_buffer(int(n))
    lib.vkpd_format_obj(*args, buf, int(n))
    return buf.raw[:n]


def write_obj(path, vertices, faces=None, lines=None, comment=None):
    with open(path, "wb") as fh:
        fh.write(format_obj(vertices, faces, lines, comment))


def write_csv(path, header, rows, chash):
    """`cli.write_csv` (`cli.py:212-217`): config hash comment, header, rows (floats as .17g)."""
    with open(path, "w") as fh:
        fh.write(f"# config {chash}\n")
        fh.write(",".join(header) + "\n")
        for row in rows:
            fh.write(",".join(_fmt(v) for v in row) + "\n")


def write_report(path, payload, chash):
    """`cli._write_report` (`cli.py:243-248`)."""
    payload = dict(payload)
    payload["config_hash"] = chash
    with open(path, "w") as fh:
        json.dump(payload, fh, indent=1, sort_keys=True)
        fh.write("\n")


def simulate_to_disk(mesh, gammas, steps, dt, out, interp, polylines, chash, forces=None, pins=(),
                     pin_path=None, colliders=(), iterations=30, damping=1.0, scenario="", solver="direct",
                     precision="fp64", tol=None):
    """The output loop of `cmd_simulate` (`cli.py:612-656`) on the device-resident step.

    interp: (n_yarn, n_nodes) sparse embedding (`transfer.v2y`); polylines: yarn vertex runs.
    Writes out/frames/mesh_NNNN.obj, yarn_NNNN.obj, out/timings.csv, out/sim_report.json;
    returns (yarn_frames (steps, n_yarn, 3), det_deviation list).  RuntimeError as pd_step.
    """
    from . import pdsolver, volmesh
    pins = np.asarray(pins, dtype=np.int64)
    timings = []

    def clock(stage, t0):
        timings.append((stage, 1000.0 * (time.perf_counter() - t0)))

    t = time.perf_counter()
    ctx = pdsolver.device_context(mesh, gammas, dt, pins, precision, tol)
    clock("assemble", t)
    t = time.perf_counter()
    ctx.set_yarn_interp(interp)
    clock("factorize", t)
    frames_dir = os.path.join(out, "frames")
    os.makedirs(frames_dir, exist_ok=True)
    tris = volmesh.boundary_faces(mesh)
    comment = f"config {chash}"
    ctx.set_state(np.asarray(mesh.nodes, dtype=float), None)
    if len(pins):
        ctx.set_pin_targets(mesh.nodes[pins] if pin_path is None else pin_path[0])
    ctx.set_colliders(colliders)
    ctx.set_forces(forces)
    n_yarn = interp.shape[0]
    yarn_frames = np.empty((steps, n_yarn, 3))
    det_dev = []
    jobs = queue.Queue(maxsize=4)
    errors = []

    def writer():
        while True:
            job = jobs.get()
            if job is None:
                return
            i, x, y, t0 = job
            try:
                write_obj(os.path.join(frames_dir, f"mesh_{i:04d}.obj"), x, faces=tris, comment=comment)
                write_obj(os.path.join(frames_dir, f"yarn_{i:04d}.obj"), y, lines=polylines, comment=comment)
            except Exception as exc:       # noqa: BLE001 - surfaced after the loop
                errors.append(exc)
            timings.append((f"write_{i:04d}", 1000.0 * (time.perf_counter() - t0)))

    th = threading.Thread(target=writer, daemon=True)
    th.start()
    try:
        for i in range(steps):
            if pin_path is not None and len(pins):
                ctx.set_pin_targets(pin_path[i])
            t = time.perf_counter()
            try:
                ctx.step(iterations, damping)
            except _abi.NonFiniteError as exc:
                raise RuntimeError(str(exc)) from None
            clock(f"step_{i:04d}", t)
            t = time.perf_counter()
            y, dd = ctx.frame_outputs(yarn=True, det=True)
            x, _ = ctx.get_state(want_v=False)
            det_dev.append(float(dd))
            yarn_frames[i] = y
            jobs.put((i, x, y, t))
    finally:
        jobs.put(None)
        th.join()
    if errors:
        raise errors[0]
    timings.sort(key=lambda r: (r[0][:4] != "asse" and r[0][:4] != "fact", r[0][-4:], r[0]))
    write_csv(os.path.join(out, "timings.csv"), ["stage", "milliseconds"], timings, chash)
    write_report(os.path.join(out, "sim_report.json"), dict(
        frames=int(steps), scenario=scenario, solver=solver,
        max_det_deviation=max(det_dev) if det_dev else 0.0, det_deviation=det_dev,
    ), chash)
    return yarn_frames, det_dev
