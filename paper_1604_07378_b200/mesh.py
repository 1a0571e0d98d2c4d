"""Tet meshes and rest-state quantities (setup; mirror of qnsim.mesh, mesh.py:1-249).

Setup runs once per scene on the host, as in the reference; the per-frame hot
path never touches these functions.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

VOLUME_EPS = 1e-14  # mesh.py:11


class MeshError(Exception):
    pass


@dataclass
class TetMesh:
    """Tetrahedral mesh, rest positions in meters (mesh.py:16-27)."""

    vertices: np.ndarray
    tets: np.ndarray
    density: float = 1000.0
    fixed: set = field(default_factory=set)

    @property
    def n(self) -> int:
        return self.vertices.shape[0]


_CUBE6 = np.array([(0, 1, 3, 7), (0, 3, 2, 7), (0, 2, 6, 7), (0, 6, 4, 7), (0, 4, 5, 7), (0, 5, 1, 7)])


@dataclass
class SpringNetwork:
    """Edge-spring discretisation of a triangle mesh (mesh.py:31-43)."""

    vertices: np.ndarray  # (n, 3)
    edges: np.ndarray  # (m, 2)
    rest_lengths: np.ndarray  # (m,)
    faces: np.ndarray  # (f, 3), for mass lumping
    density: float = 1.0  # kg/m^2 (areal)
    fixed: set = field(default_factory=set)

    @property
    def n(self) -> int:
        return self.vertices.shape[0]


def load_obj_springs(path, density: float = 1.0) -> SpringNetwork:
    """OBJ triangle mesh as a spring network: unique triangle edges, sorted
    (mesh.py:135-171)."""
    try:
        with open(path) as fh:
            raw = fh.readlines()
    except OSError as exc:
        raise MeshError(f"cannot read {path}: {exc}") from exc
    verts, faces = [], []
    for lineno, line in enumerate(raw, 1):
        text = line.split("#", 1)[0].strip()
        if not text:
            continue
        parts = text.split()
        if parts[0] == "v":
            try:
                verts.append([float(parts[1]), float(parts[2]), float(parts[3])])
            except (ValueError, IndexError) as exc:
                raise MeshError(f"{path}:{lineno}: bad vertex record {text!r}") from exc
        elif parts[0] == "f":
            try:
                faces.append([int(p.split("/")[0]) - 1 for p in parts[1:4]])
            except (ValueError, IndexError) as exc:
                raise MeshError(f"{path}:{lineno}: bad face record {text!r}") from exc
    if not verts or not faces:
        raise MeshError(f"{path}: no triangles found")
    vertices = np.asarray(verts)
    faces = np.asarray(faces, dtype=np.int64)
    if faces.min() < 0 or faces.max() >= vertices.shape[0]:
        raise MeshError(f"{path}: face index out of range")
    edge_set = set()
    for tri in faces:
        for a, b in ((tri[0], tri[1]), (tri[1], tri[2]), (tri[0], tri[2])):
            edge_set.add((min(a, b), max(a, b)))
    edges = np.asarray(sorted(edge_set), dtype=np.int64)
    rest = np.linalg.norm(vertices[edges[:, 1]] - vertices[edges[:, 0]], axis=1)
    if np.any(rest <= 0):
        raise MeshError(f"{path}: zero-length edge in mesh")
    return SpringNetwork(vertices=vertices, edges=edges, rest_lengths=rest, faces=faces, density=float(density))


def grid_bar(nx, ny, nz, size):
    """Freudenthal 6-tet bar, vectorised (same ids and orientation as
    qnsim.assets.bar_mesh, assets.py:10-69): vertex (i, j, k) has id
    (i (ny+1) + j)(nz+1) + k; cell corners are coded di*4 + dj*2 + dk."""
    sx, sy, sz = size[0] / nx, size[1] / ny, size[2] / nz
    verts = grid_bar_verts(nx, ny, nz, size)
    ci, cj, ck = (a.ravel() for a in np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"))
    corner = np.stack([((ci + (c >> 2)) * (ny + 1) + (cj + ((c >> 1) & 1))) * (nz + 1) + (ck + (c & 1))
                       for c in range(8)], axis=1)
    tets = corner[:, _CUBE6].reshape(-1, 4).astype(np.int64)
    e = verts[tets[:, 1:]] - verts[tets[:, :1]]
    flip = np.linalg.det(e) < 0
    tets[flip] = tets[flip][:, [0, 1, 3, 2]]
    return verts, tets


def grid_bar_verts(nx, ny, nz, size):
    """Rest vertices of grid_bar (vertex (i, j, k) at (i sx, j sy, k sz))."""
    sx, sy, sz = size[0] / nx, size[1] / ny, size[2] / nz
    ii, jj, kk = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), np.arange(nz + 1), indexing="ij")
    return np.column_stack([0.0 + ii.ravel() * sx, 0.0 + jj.ravel() * sy, 0.0 + kk.ravel() * sz])


def grid_bar_cells(nx, ny, nz, size, c_lo, c_hi):
    """Tets of the cells with x index in [c_lo, c_hi) of grid_bar(nx, ny, nz,
    size), global vertex ids, in grid_bar's order (the cells of an x range are
    a contiguous block of its tet array), without building the whole mesh."""
    sx, sy, sz = size[0] / nx, size[1] / ny, size[2] / nz
    ci, cj, ck = (a.ravel() for a in np.meshgrid(np.arange(c_lo, c_hi), np.arange(ny), np.arange(nz), indexing="ij"))
    corner = np.stack([((ci + (c >> 2)) * (ny + 1) + (cj + ((c >> 1) & 1))) * (nz + 1) + (ck + (c & 1))
                       for c in range(8)], axis=1)
    tets = corner[:, _CUBE6].reshape(-1, 4).astype(np.int64)
    plane = (ny + 1) * (nz + 1)
    g = tets - c_lo * plane  # local grid coordinates of the corners (rest, unjittered)
    k = g % (nz + 1)
    j = (g // (nz + 1)) % (ny + 1)
    i = g // plane + c_lo
    p = np.stack([i * sx, j * sy, k * sz], axis=-1).astype(np.float64)
    e = p[:, 1:] - p[:, :1]
    flip = np.linalg.det(e) < 0
    tets[flip] = tets[flip][:, [0, 1, 3, 2]]
    return tets


def bar_mesh(nx=12, ny=4, nz=4, size=(1.5, 0.5, 0.5)):
    """assets.bar_mesh signature (assets.py:66-69)."""
    return grid_bar(nx, ny, nz, size)


def tet_volumes(mesh: TetMesh) -> np.ndarray:
    v = mesh.vertices[mesh.tets]
    return np.linalg.det(v[:, 1:] - v[:, :1]) / 6.0


def lumped_masses(mesh) -> np.ndarray:
    """rho V / 4 to each tet corner, or rho A / 3 to each triangle corner of a
    spring network (mesh.py:176-197)."""
    m = np.zeros(mesh.n)
    if isinstance(mesh, SpringNetwork):
        v = mesh.vertices[mesh.faces]
        areas = 0.5 * np.linalg.norm(np.cross(v[:, 1] - v[:, 0], v[:, 2] - v[:, 0]), axis=1)
        share = mesh.density * areas / 3.0
        for c in range(3):
            np.add.at(m, mesh.faces[:, c], share)
    else:
        share = mesh.density * tet_volumes(mesh) / 4.0
        for c in range(4):
            np.add.at(m, mesh.tets[:, c], share)
    bad = np.nonzero(m <= 0)[0]
    if bad.size:
        raise MeshError(f"vertex {bad[0]} has zero mass (isolated vertex?)")
    return m


def tet_diff_operators(mesh: TetMesh):
    """G (m,4,3): G[1:] = Dm^-1, G[0] = -sum; rest volumes (mesh.py:200-216)."""
    v = mesh.vertices[mesh.tets]
    Dm = np.swapaxes(v[:, 1:] - v[:, :1], 1, 2)
    vols = np.linalg.det(Dm) / 6.0
    if np.any(vols < VOLUME_EPS):
        raise MeshError("degenerate rest tet in diff-operator construction")
    inv = np.linalg.inv(Dm)
    G = np.empty((mesh.tets.shape[0], 4, 3))
    G[:, 1:, :] = inv
    G[:, 0, :] = -inv.sum(axis=1)
    return G, vols


def _rows(path):
    try:
        with open(path) as fh:
            raw = fh.readlines()
    except OSError as exc:
        raise MeshError(f"cannot read {path}: {exc}") from exc
    out = [ln.split("#", 1)[0].split() for ln in raw]
    out = [r for r in out if r]
    if not out:
        raise MeshError(f"{path}: file contains no data")
    return out


def load_tet_mesh(node_file, ele_file, density: float) -> TetMesh:
    """TetGen .node/.ele reader: 0/1-based ids, orientation fix (mesh.py:52-68)."""
    nr = _rows(node_file)
    nv = int(nr[0][0])
    if len(nr) - 1 < nv:
        raise MeshError(f"{node_file}: expected {nv} vertex rows, found {len(nr) - 1}")
    try:
        base = 0 if int(nr[1][0]) == 0 else 1
        verts = np.array([[float(r[1]), float(r[2]), float(r[3])] for r in nr[1:1 + nv]])
    except (ValueError, IndexError) as exc:
        raise MeshError(f"{node_file}: bad vertex row") from exc
    er = _rows(ele_file)
    ne = int(er[0][0])
    if len(er) - 1 < ne:
        raise MeshError(f"{ele_file}: expected {ne} element rows, found {len(er) - 1}")
    try:
        tets = np.array([[int(p) for p in r[1:5]] for r in er[1:1 + ne]], dtype=np.int64) - base
    except (ValueError, IndexError) as exc:
        raise MeshError(f"{ele_file}: bad element row") from exc
    if tets.min() < 0 or tets.max() >= nv:
        raise MeshError(f"{ele_file}: element index out of range [0, {nv})")
    if nv < 4:
        raise MeshError(f"{node_file}: tet mesh needs at least 4 vertices")
    mesh = TetMesh(verts, tets, float(density))
    vols = tet_volumes(mesh)
    flip = vols < 0
    tets[flip] = tets[flip][:, [0, 1, 3, 2]]
    bad = np.nonzero(np.abs(vols) < VOLUME_EPS)[0]
    if bad.size:
        raise MeshError(f"{ele_file}: tet {bad[0]} has zero volume")
    return mesh
