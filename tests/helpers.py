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
