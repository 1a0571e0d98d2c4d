"""Output formats of the reference harness: the
convergence CSV consumed by its plotter and per-frame OBJ surfaces.

Host-side file writers only (no simulation arithmetic): `write_csv` follows
harness.py:36,390-399 (schema `frame,iteration,g,rel_error,ls_trials,cum_ms`,
`g` and `rel_error` at %.17g, `cum_ms` at %.3f), `export_frames` follows
harness.py:408-420, `surface_triangles` mesh.py:236-249.
"""

from __future__ import annotations

import os

import numpy as np

from paper_1604_07378_b200.mesh import SpringNetwork

CSV_HEADER = "frame,iteration,g,rel_error,ls_trials,cum_ms"


def write_csv(path, records):
    """One row per (frame, iteration) of a list of ConvergenceRecords."""
    os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
    lines = [CSV_HEADER]
    for frame, rec in enumerate(records):
        for it, g in enumerate(rec.g):
            rel = f"{rec.rel_error[it]:.17g}" if rec.rel_error else ""
            lines.append(f"{frame},{it + 1},{g:.17g},{rel},{rec.ls_trials[it]},{rec.cum_ms[it]:.3f}")
    with open(path, "w") as fh:
        fh.write("\n".join(lines) + "\n")


def surface_triangles(mesh) -> np.ndarray:
    """Faces referenced by exactly one tet, outward for positively oriented
    tets, sorted (the reference's faces of each tet: (0,2,1) (0,1,3) (0,3,2) (1,2,3))."""
    t = np.asarray(mesh.tets, dtype=np.int64)
    tris = np.concatenate([t[:, [0, 2, 1]], t[:, [0, 1, 3]], t[:, [0, 3, 2]], t[:, [1, 2, 3]]])
    key = np.sort(tris, axis=1)
    _, inv, cnt = np.unique(key, axis=0, return_inverse=True, return_counts=True)
    once = cnt[inv.ravel()] == 1
    out = tris[once]
    order = np.lexsort(out.T[::-1])
    return out[order]


def mesh_faces(mesh):
    return mesh.faces if isinstance(mesh, SpringNetwork) else surface_triangles(mesh)


def export_frames(states, directory, faces):
    """frame_0000.obj, frame_0001.obj, ...: vertices at %.12g, 1-based faces."""
    os.makedirs(directory, exist_ok=True)
    paths = []
    for i, x in enumerate(states):
        path = os.path.join(directory, f"frame_{i:04d}.obj")
        body = [f"v {vx:.12g} {vy:.12g} {vz:.12g}" for vx, vy, vz in np.asarray(x)]
        body += [f"f {a + 1} {b + 1} {c + 1}" for a, b, c in np.asarray(faces)]
        with open(path, "w") as fh:
            fh.write("\n".join(body) + "\n")
        paths.append(path)
    return paths
