"""Shared test helpers: golden loading, oracle material construction, the
bar_twist_small scene of the reference's golden CSVs (harness.py:246-344)."""
import csv
import json
import os

import numpy as np

import oracle.qnsim_oracle as O
from paper_1604_07378_b200 import scenes

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FIX = os.path.join(GOLDEN, "ref_fixtures")


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def oracle_material(spec):
    f = {"zero": lambda s: O.Zero(), "poly": lambda s: O.Poly(s[1]), "log": lambda s: O.Log(s[1], s[2]),
         "hermite": lambda s: O.Hermite(s[1])}
    return O.VLMaterial(*[f[x[0]](x) for x in spec])


def read_csv(path):
    with open(path) as fh:
        rows = list(csv.DictReader(fh))
    frames = max(int(r["frame"]) for r in rows) + 1
    its = max(int(r["iteration"]) for r in rows)
    g = np.zeros((frames, its))
    tr = np.zeros((frames, its), dtype=int)
    for r in rows:
        g[int(r["frame"]), int(r["iteration"]) - 1] = float(r["g"])
        tr[int(r["frame"]), int(r["iteration"]) - 1] = int(r["ls_trials"])
    return g, tr


class TwistScene:
    """bar_twist_small.json (NH mu=1e5, lambda=4e5; x=0 face fixed; x=0.6 face
    twisted at 180 deg/s about x through (0, 0.1, 0.1)), as driven by the
    reference harness for the golden CSVs: 40 frames x 20 iterations."""

    frames = 40
    iterations = 20

    def __init__(self):
        with open(os.path.join(FIX, "bar_twist_small.json")) as fh:
            scn = json.load(fh)
        self.verts, self.tets = O.read_node_ele(os.path.join(FIX, "bar_small.node"), os.path.join(FIX, "bar_small.ele"))
        self.h = float(scn["h"])
        self.gravity = tuple(scn["gravity"])
        self.density = float(scn["mesh"]["density"])
        self.mu, self.lam = float(scn["material"]["mu"]), float(scn["material"]["lambda"])
        groups = []
        for sel in scn["fixed"]:
            lo, hi = np.asarray(sel["box"][0]), np.asarray(sel["box"][1])
            idx = np.nonzero(np.all((self.verts >= lo) & (self.verts <= hi), axis=1))[0]
            groups.append((idx, sel.get("motion")))
        self.groups = groups
        self.fixed = np.asarray(sorted(set(int(i) for g, _ in groups for i in g)), dtype=np.int64)

    def targets(self, frame):
        t = (frame + 1) * self.h
        pos = {int(i): self.verts[i].copy() for i in self.fixed}
        for idx, motion in self.groups:
            if motion is None:
                continue
            p = O.twist_targets(self.verts, idx, motion["axis"], motion["center"], motion["degrees_per_second"], t)
            for k, v in enumerate(idx):
                pos[int(v)] = p[k]
        return np.array([pos[int(i)] for i in self.fixed])


def material_specs():
    """Material cases shared by the golden generator and the tests."""
    return {
        "neohookean": scenes.builtin_spec("neohookean", 1e5, 4e5),
        "stvk": scenes.builtin_spec("stvk", *scenes.lame(1e6, 0.4)),
        "polynomial": scenes.builtin_spec("polynomial", 2e4),
        "corotated": scenes.builtin_spec("corotated", 1e4, 4e4),
        "mooney_rivlin": scenes.builtin_spec("mooney_rivlin", mu1=3e4, mu2=1e4, lam=2e5),
        "spline": scenes.nh_spline_spec(np.random.default_rng(11)),
        "poly_cubic": scenes.c5(grid=(2, 1, 1)).material,
    }


def collider_bar_scene():
    """A c1-style NH bar (10x3x3, x=0 face pinned) thrown down (v0 = -2 m/s in
    z) onto a half-space, a sphere and a torus: every collider kind of
    dynamics.py:199-270 is active within the first frames.  Collider specs:
    (kind, ...) tuples, built by the caller for each implementation."""
    sc = scenes.c1(grid=(10, 3, 3), iterations=10)
    v0 = np.zeros_like(sc.verts)
    v0[:, 2] = -2.0
    v0[sc.fixed] = 0.0
    sc.q_prev = sc.q_l - sc.h * v0
    cols = [("halfspace", (0.0, 0.0, -0.08), (0.0, 0.1, 1.0)),
            ("sphere", (0.75, 0.15, -0.25), 0.27),
            ("torus", (0.35, 0.15, -0.16), 0.2, 0.12)]
    return sc, cols


def make_colliders(cols, ns):
    """Collider objects of module `ns` (oracle: HalfSpace/Sphere/Torus;
    package dynamics: HalfSpace/SphereCollider/TorusCollider)."""
    sphere = getattr(ns, "SphereCollider", None) or ns.Sphere
    torus = getattr(ns, "TorusCollider", None) or ns.Torus
    out = []
    for c in cols:
        if c[0] == "halfspace":
            out.append(ns.HalfSpace(c[1], c[2]))
        elif c[0] == "sphere":
            out.append(sphere(c[1], c[2]))
        else:
            out.append(torus(c[1], c[2], c[3]))
    return out


class SphereDropScene:
    """The reference's sphere_drop.json (corotated sphere mesh dropped on a
    half-space, collision_weight 3e5, 20 iterations), as run by its harness
    for tests/golden/frames_sphere_drop.npz."""

    def __init__(self):
        with open(os.path.join(FIX, "sphere_drop.json")) as fh:
            scn = json.load(fh)
        self.verts, self.tets = O.read_node_ele(os.path.join(FIX, "sphere.node"), os.path.join(FIX, "sphere.ele"))
        self.h = float(scn["h"])
        self.gravity = tuple(scn["gravity"])
        self.density = float(scn["mesh"]["density"])
        self.material = scenes.builtin_spec("corotated", float(scn["material"]["mu"]), float(scn["material"]["lambda"]))
        self.iterations = int(scn["solver"]["iterations"])
        self.m = int(scn["solver"].get("m", 5))
        self.collision_weight = float(scn["collision_weight"])
        self.cols = [("halfspace", tuple(c["point"]), tuple(c["normal"])) for c in scn["colliders"]]
        self.fixed = np.zeros(0, dtype=np.int64)
        self.q_l = self.verts.copy()
        self.q_prev = self.verts.copy()


class ClothScene:
    """The reference's cloth_hang.json: cloth20.obj as a mass-spring network
    (k = 200, areal density 0.2), corners 0 and 19 pinned, lbfgs 10 its."""

    def __init__(self):
        with open(os.path.join(FIX, "cloth_hang.json")) as fh:
            scn = json.load(fh)
        self.verts, self.edges, self.rest, self.faces = O.read_obj_springs(os.path.join(FIX, "cloth20.obj"))
        self.density = float(scn["mesh"]["density"])
        self.k = float(scn["material"]["k"])
        self.h = float(scn["h"])
        self.gravity = tuple(scn["gravity"])
        self.fixed = np.asarray(scn["fixed"][0]["indices"], dtype=np.int64)
        self.iterations = int(scn["solver"]["iterations"])
        self.m = 5
        self.q_l = self.verts.copy()
        self.q_prev = self.verts.copy()


def aniso_cases(m):
    """Fibre assignments of tests/golden/frames_aniso.npz (make_golden.gen_aniso)."""
    return {"uniform": [(e, (1.0, 0.2, 0.0), 3e5) for e in range(m)],
            "two": [(e, (1.0, 0.0, 1.0) if e % 2 else (0.0, 1.0, 0.5), 1e5 if e % 2 else 4e5) for e in range(m)]}
