"""Accept the reference's own objects at the drop-in boundary.

A caller of `qnsim` (e.g. `qnsim.harness.SimulationRun`, harness.py:288-351)
builds its mesh, materials, fit interval and colliders with `qnsim` classes and
then calls `build_system` / `simulate_frame`.  When those two names are swapped
for this package's, the inputs are still `qnsim` objects, so
`build_system` converts them here — by class name and public attributes, with no
import of `qnsim` — into this package's types:

* `qnsim.mesh.TetMesh` / `SpringNetwork` (mesh.py:16-43)
* `qnsim.materials.MaterialModel` with ZeroFn / PolyFn / LogFn / HermiteFn
  scalar functions (materials.py:32-159, keeping a cached `k_fit`),
  `PDMaterial` (:163-173), `FitInterval` (:137-143), and group assignments
  `[(tet_ids, material), ...]` (dynamics.py:330-345)
* `qnsim.dynamics.HalfSpace` / `SphereCollider` / `TorusCollider`
  (dynamics.py:199-270)

Objects that already are this package's types pass through unchanged.
"""

from __future__ import annotations

import numpy as np

from paper_1604_07378_b200 import materials as M
from paper_1604_07378_b200 import mesh as ME


def _cls(obj) -> str:
    return type(obj).__name__


def scalar_fn(f):
    if isinstance(f, (M.ZeroFn, M.PolyFn, M.LogFn, M.HermiteFn, M.SqDevFn)):
        return f
    name = _cls(f)
    if name == "ZeroFn":
        return M.ZeroFn()
    if name == "PolyFn":
        return M.PolyFn(np.asarray(f.coeffs, dtype=np.float64))
    if name == "LogFn":
        return M.LogFn(f.alpha, f.beta, f.eps)
    if name == "HermiteFn":
        return M.HermiteFn(np.stack([f.xs, f.ys, f.ts], axis=1))
    raise M.MaterialError(f"cannot adopt scalar function {name}")


def material(m):
    if isinstance(m, (M.MaterialModel, M.PDMaterial)):
        return m
    name = _cls(m)
    if name == "MaterialModel":
        out = M.MaterialModel(scalar_fn(m.a), scalar_fn(m.b), scalar_fn(m.c), getattr(m, "name", "custom"))
        k = getattr(m, "k_fit", None)
        if k is not None:
            out.k_fit = float(k)
        return out
    if name == "PDMaterial":
        return M.PDMaterial(m.kind, float(m.k))
    raise M.MaterialError(f"cannot adopt material {name}")


def materials(ms):
    """A material or a group assignment [(tet_ids, material), ...]."""
    if isinstance(ms, (list, tuple)):
        return [(idx, material(m)) for idx, m in ms]
    return material(ms)


def fit_interval(iv):
    if isinstance(iv, M.FitInterval):
        return iv
    return M.FitInterval(float(iv.x_start), float(iv.x_end))


def mesh(msh):
    if isinstance(msh, (ME.TetMesh, ME.SpringNetwork)):
        return msh
    name = _cls(msh)
    if name == "TetMesh":
        return ME.TetMesh(np.asarray(msh.vertices, dtype=np.float64), np.asarray(msh.tets),
                          float(msh.density), set(getattr(msh, "fixed", set())))
    if name == "SpringNetwork":
        return ME.SpringNetwork(np.asarray(msh.vertices, dtype=np.float64), np.asarray(msh.edges),
                                np.asarray(msh.rest_lengths, dtype=np.float64), np.asarray(msh.faces),
                                float(msh.density), set(getattr(msh, "fixed", set())))
    raise TypeError(f"cannot adopt mesh {name}")


def collider(c):
    from paper_1604_07378_b200 import dynamics as D
    if isinstance(c, (D.HalfSpace, D.SphereCollider, D.TorusCollider)):
        return c
    name = _cls(c)
    if name == "HalfSpace":
        return D.HalfSpace(c.point, c.normal)
    if name == "SphereCollider":
        return D.SphereCollider(c.center, c.radius)
    if name == "TorusCollider":
        return D.TorusCollider(c.center, c.R, c.r)
    raise TypeError(f"cannot adopt collider {name}")
