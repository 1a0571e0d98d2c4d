"""configs[4] goldens from the UNMODIFIED reference with one substitution
(SURVEY.md §8c): `sysfact` is CPU conjugate gradients on A_free to a relative
residual of 1e-13 (oracle.qnsim_oracle.CGFactor / oracle/cg_free.c) instead of
the dense Cholesky, which cannot be formed at 12 M dofs.

    python tests/golden/make_c5_golden.py [--grid 400 100 100] [--frames 2] [--out frames_c5_full.npz]

Everything else is the reference's own code: `qnsim.dynamics.build_system`
(dynamics.py:351-434: masses, tet groups, the COO->CSR assembly of L and A,
free/fixed sets, scale) runs as shipped, with two calls intercepted for the
duration of the build: `A.toarray()` (dynamics.py:413) returns a view that
hands `A[np.ix_(free, free)]` back as the sparse A_free, and `factorize_spd`
(:414) returns the CG solver.  `qnsim.solvers.simulate_frame` (solvers.py:260-352,
VLGroup energy / gradient, svd_rv_batch, Armijo) then runs unmodified through
`solve_prefactored(sysfact, B)` = `sysfact.solve(B)` (linalg.py:57-59).

Stored per frame (frames 1..F from the scene's initial state): g0, the
per-iteration g / ls_trials / alphas, stagnated, the CG iteration counts and
true residuals of every solve, positions of sampled vertices (seeded random
ids + the free end face), and size-independent checks of the whole position
array (max |x|, the seeded linear functional w.x, ||x - rest||).  Run in the
build container (needs /root/reference); the full 400x100x100 bar takes a few
hours on one core (the reference's element passes are single-threaded numpy).
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np
import scipy.sparse

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

from qnsim import dynamics as ref_dyn  # noqa: E402
from qnsim import mesh as ref_mesh  # noqa: E402
from qnsim import solvers as ref_solvers  # noqa: E402

import oracle.qnsim_oracle as O  # noqa: E402
from paper_1604_07378_b200 import scenes  # noqa: E402
from tests.golden.make_golden import ref_material  # noqa: E402

SAMPLE_SEED = 7
SAMPLE_RANDOM = 4096
FUNCTIONAL_SEED = 11


def sample_ids(grid, n):
    rng = np.random.default_rng(SAMPLE_SEED)
    end = scenes.face_ids(*grid, grid[0])
    return np.unique(np.concatenate([rng.choice(n, size=min(SAMPLE_RANDOM, n), replace=False), end]))


def functional(n):
    return np.random.default_rng(FUNCTIONAL_SEED).standard_normal((n, 3))


class _LazyDense:
    """Stands in for `A.toarray()` (dynamics.py:413): indexing it with
    np.ix_(free, free) returns the sparse A_free."""

    def __init__(self, A):
        self.A = A.tocsr()

    def __getitem__(self, key):
        rows, cols = key
        return self.A[np.asarray(rows).ravel()][:, np.asarray(cols).ravel()].tocsr()


def build_reference_system(sc):
    mesh = ref_mesh.TetMesh(vertices=sc.verts, tets=sc.tets, density=sc.density)
    mat = ref_material(sc.material)
    saved = (scipy.sparse.csr_matrix.toarray, ref_dyn.factorize_spd)
    scipy.sparse.csr_matrix.toarray = lambda self, *a, **k: _LazyDense(self)
    ref_dyn.factorize_spd = lambda A: O.CGFactor(A, tol=1e-13)
    try:
        system = ref_dyn.build_system(mesh, mat, h=sc.h, gravity=sc.gravity, fixed=sc.fixed)
    finally:
        scipy.sparse.csr_matrix.toarray, ref_dyn.factorize_spd = saved
    return system


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, nargs=3, default=[400, 100, 100])
    ap.add_argument("--frames", type=int, default=2)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    grid = tuple(a.grid)
    out = a.out or os.path.join(HERE, "frames_c5_%dx%dx%d.npz" % grid)
    sc = scenes.c5(grid=grid)
    t0 = time.time()
    system = build_reference_system(sc)
    print(f"built {grid}: n={sc.verts.shape[0]} m={sc.tets.shape[0]} n_free={system.free.size} "
          f"nnz(A_free)={system.sysfact.val.size} in {time.time() - t0:.0f} s", flush=True)
    n = sc.verts.shape[0]
    ids = sample_ids(grid, n)
    w = functional(n)
    cfg = ref_solvers.SolverConfig(kind="lbfgs", iterations=sc.iterations, m=sc.m)
    st = ref_dyn.SimState(q_l=np.array(sc.q_l), q_prev=np.array(sc.q_prev))
    res = {"grid": np.array(grid), "frames": a.frames, "ids": ids, "iterations": sc.iterations, "m": sc.m,
           "cg_tol": 1e-13}
    for f in range(a.frames):
        t = time.time()
        nlog = len(system.sysfact.log)
        st, rec = ref_solvers.simulate_frame(system, st, cfg)
        x = st.q_l
        res[f"g0_{f}"] = rec.g0
        res[f"g_{f}"] = np.array(rec.g)
        res[f"trials_{f}"] = np.array(rec.ls_trials)
        res[f"alphas_{f}"] = np.array(rec.alphas)
        res[f"stagnated_{f}"] = rec.stagnated
        res[f"x_{f}"] = x[ids]
        res[f"xmax_{f}"] = np.abs(x).max()
        res[f"wx_{f}"] = float(np.vdot(w, x))
        res[f"disp_{f}"] = float(np.linalg.norm(x - sc.verts))
        log = system.sysfact.log[nlog:]
        res[f"cg_iters_{f}"] = np.array([l[0] for l in log])
        res[f"cg_relres_{f}"] = np.array([l[1] for l in log])
        res["frames"] = f + 1
        print(f"frame {f}: {time.time() - t:.0f} s, g {rec.g[-1]:.17g}, trials {rec.ls_trials}, "
              f"cg its {[l[0][0] for l in log]}, max relres {np.max([l[1] for l in log]):.2e}", flush=True)
        np.savez_compressed(out, **res)
    print("wrote", out)


if __name__ == "__main__":
    main()
