"""CPU-side checks: the C-ABI library builds, loads and exports every symbol
declared in include/qnsim_b200.h with matching struct layouts; host logic
(scene generation, material packing, the host supernodal factorisation and a
CPU replay of the device solve algorithm) — no GPU compute calls."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import oracle.qnsim_oracle as O
from paper_1604_07378_b200 import _lib, materials, scenes
from tests.helpers import oracle_material

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "qnsim_b200.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(qn_\w+)\(", text, flags=re.M)))


def test_library_builds_and_exports_every_declared_symbol(built_lib):
    lib = _lib.load(built_lib)
    names = declared_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", built_lib], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (qn_\w+)", out))
    assert set(names) <= exported
    assert set(_lib.SIGNATURES) | {"qn_last_error"} == set(names)


def test_struct_layouts_match_c(tmp_path):
    src = tmp_path / "layout.c"
    src.write_text("""
#include <stdio.h>
#include <stddef.h>
#include "qnsim_b200.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu %zu\\n", sizeof(qn_scalar_fn), sizeof(qn_material), sizeof(qn_system_desc),
         offsetof(qn_system_desc, h), offsetof(qn_system_desc, free_coords), sizeof(qn_solver_config),
         sizeof(qn_frame_record), sizeof(qn_factor_info));
  return 0;
}
""")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", f"-I{ROOT}/include", str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    want = [C.sizeof(_lib.ScalarFn), C.sizeof(_lib.Material), C.sizeof(_lib.SystemDesc),
            _lib.SystemDesc.h.offset, _lib.SystemDesc.free_coords.offset, C.sizeof(_lib.SolverConfigC),
            C.sizeof(_lib.FrameRecord), C.sizeof(_lib.FactorInfo)]
    assert got == want


def test_no_device_means_loud_failure(built_lib):
    if _lib.device_count() > 0:
        pytest.skip("GPU present")
    with pytest.raises(_lib.QnRuntimeError):
        _lib.require_gpu()


@pytest.fixture(scope="module")
def hostcheck(tmp_path_factory):
    out = tmp_path_factory.mktemp("hc") / "libhc.so"
    subprocess.run(["g++", "-O2", "-fopenmp", "-std=c++17", "-fPIC", "-shared", f"-I{ROOT}/include",
                    f"-I{ROOT}/paper_1604_07378_b200/csrc", "-I/usr/local/cuda/include", "-o", str(out),
                    f"{ROOT}/tests/native/factor_hostcheck.cpp", f"{ROOT}/paper_1604_07378_b200/csrc/qn_factor.cpp",
                    f"{ROOT}/paper_1604_07378_b200/csrc/qn_amg.cpp"],
                   check=True)
    lib = C.CDLL(str(out))
    lib.hc_last_error.restype = C.c_char_p
    return lib


def _hc_solve(lib, A, coords, B, values=None, nbatch=1, b=0):
    A = A.tocsr()
    A.sort_indices()
    n = A.shape[0]
    X = np.zeros((n, 3))
    st = np.zeros(8, dtype=np.int64)
    vals = np.ascontiguousarray(A.data if values is None else values)
    rc = lib.hc_factor_solve(C.c_int64(n), _lib.ptr(_lib.i64(A.indptr)), _lib.ptr(_lib.i32(A.indices)),
                             _lib.ptr(vals), C.c_int64(nbatch), _lib.ptr(coords), C.c_int64(b), _lib.ptr(B),
                             _lib.ptr(X), _lib.ptr(st))
    return rc, X, st


@pytest.mark.parametrize("cfg", ["c1", "c2"])
def test_host_supernodal_factor_and_solve_replay(hostcheck, cfg):
    sc = scenes.CONFIGS[cfg](frames=1)
    osys = O.build(sc.verts, sc.tets, sc.density, oracle_material(sc.material), sc.h, sc.gravity, sc.fixed)
    B = np.random.default_rng(0).standard_normal((osys.free.size, 3))
    rc, X, st = _hc_solve(hostcheck, osys.A_free, _lib.f64(sc.verts[osys.free]), B)
    assert rc == 0
    ref = osys.factor.solve(B)
    assert np.abs(X - ref).max() <= 1e-12 * np.abs(ref).max()
    nsup, nnz_l, depth, max_rows, nft, nbt, ktop = st[:7]
    if cfg == "c1":  # small system: the whole tree is the dense top (one product)
        assert nft == 0 and nbt == 0 and ktop == osys.free.size
    else:  # narrow separators (16x16 planes): sparse tasks all the way up
        assert ktop == 0 and nft > 0 and nbt > 0
    assert depth <= 16  # nested dissection + amalgamation keep the dependency tree shallow
    if cfg == "c2":
        assert nnz_l < 3.34e6  # below the SuperLU-MMD fill of the survey probe


def test_host_partial_dense_top_replay(hostcheck, monkeypatch):
    # force the dense top onto c2's narrow top levels (the path c3 takes by default)
    monkeypatch.setenv("QN_TOP_MIN_WIDTH", "0")
    sc = scenes.c2(frames=1)
    osys = O.build(sc.verts, sc.tets, sc.density, oracle_material(sc.material), sc.h, sc.gravity, sc.fixed)
    B = np.random.default_rng(2).standard_normal((osys.free.size, 3))
    rc, X, st = _hc_solve(hostcheck, osys.A_free, _lib.f64(sc.verts[osys.free]), B)
    assert rc == 0
    ref = osys.factor.solve(B)
    assert np.abs(X - ref).max() <= 1e-12 * np.abs(ref).max()
    ktop, nft = st[6], st[4]
    assert 0 < ktop <= 4096 and nft > 0


def test_host_factor_batch_and_not_spd(hostcheck):
    sc = scenes.c1()
    osys = O.build(sc.verts, sc.tets, sc.density, oracle_material(sc.material), sc.h, sc.gravity, sc.fixed)
    A = osys.A_free.tocsr()
    A.sort_indices()
    vals = np.concatenate([A.data, 2.0 * A.data])
    B = np.random.default_rng(1).standard_normal((A.shape[0], 3))
    rc, X1, _ = _hc_solve(hostcheck, A, _lib.f64(sc.verts[osys.free]), B, values=vals, nbatch=2, b=1)
    assert rc == 0
    ref = osys.factor.solve(B) / 2.0
    assert np.abs(X1 - ref).max() <= 1e-12 * np.abs(ref).max()
    import scipy.sparse as sp
    bad = sp.csr_matrix(np.diag([1.0, -2.0, 3.0]))
    rc, _, _ = _hc_solve(hostcheck, bad, None, np.ones((3, 3)))
    assert rc == _lib.QN_ERR_NOT_SPD
    assert b"not positive definite" in hostcheck.hc_last_error()


def test_scene_generation_shapes():
    s1 = scenes.c1()
    assert s1.tets.shape == (3000, 4) and s1.verts.shape == (756, 3) and s1.fixed.size == 36
    s2 = scenes.c2()
    assert s2.tets.shape == (81000, 4) and s2.verts.shape == (15616, 3) and s2.fixed.size == 256
    assert np.abs(s2.q_prev - s2.q_l)[s2.fixed].max() == 0
    s3 = scenes.c3(grid=(10, 4, 4))
    assert s3.fixed.size == 2 * 25
    mid = np.abs(s3.verts[:, 0] - 0.5).argmin()
    assert np.linalg.norm(s3.q_l - s3.verts, axis=1).max() == pytest.approx(0.2, rel=0.05)
    s4 = scenes.c4(instances=8)
    assert s4.q_l.shape == (8, 756, 3) and len(s4.batch_materials) == 8
    s5 = scenes.c5(grid=(8, 2, 2))
    assert s5.material[0][0] == "poly" and len(s5.material[0][1]) == 7
    # seeded: identical inputs on every call
    np.testing.assert_array_equal(scenes.c1().verts, s1.verts)


def test_material_packing_and_setup_functions():
    for spec in (scenes.builtin_spec("neohookean", 1e5, 4e5), scenes.nh_spline_spec(np.random.default_rng(0)),
                 scenes.c5(grid=(2, 1, 1)).material):
        mat = materials.from_spec(spec)
        om = oracle_material(spec)
        assert mat.shift == om.shift
        assert materials.estimate_stiffness(mat) == O.fit_stiffness(om)
        c = mat.to_c()
        for f, s in ((c.a, spec[0]), (c.b, spec[1]), (c.c, spec[2])):
            assert f.kind == {"zero": 0, "poly": 1, "log": 2, "hermite": 3}[s[0]]
    with pytest.raises(materials.MaterialError):
        materials.make_builtin("unobtainium")
    with pytest.raises(materials.MaterialError):
        materials.make_builtin("neohookean", {"mu": -1})
    with pytest.raises(materials.MaterialError):
        materials.PolyFn(np.ones(20))


def test_solver_config_validation():
    from paper_1604_07378_b200.solvers import SolverConfig, SolverError
    SolverConfig()
    for kw in (dict(kind="steepest"), dict(gamma=1.5), dict(gamma=0.0), dict(rho=1.0), dict(m=-1),
               dict(iterations=0), dict(lbfgs_init="bogus")):
        with pytest.raises(SolverError):
            SolverConfig(**kw)
    c = SolverConfig(kind="lbfgs", iterations=7, m=3).to_c()
    assert (c.kind, c.iterations, c.m, c.line_search) == (1, 7, 3, 1)
    with pytest.raises(NotImplementedError):
        SolverConfig(kind="newton").to_c()


def test_host_amg_pcg_on_scaled_c5(hostcheck):
    """Smoothed-aggregation AMG hierarchy + the host mirror of the device
    V(1,1)-preconditioned CG: converges to 1e-10 in few iterations and agrees
    with a direct solve."""
    import scipy.sparse.linalg as spla
    sc = scenes.c5(grid=(40, 10, 10))
    osys = O.build(sc.verts, sc.tets, sc.density, oracle_material(sc.material), sc.h, sc.gravity, sc.fixed)
    A = osys.A_free.tocsr()
    A.sort_indices()
    n = A.shape[0]
    B = np.random.default_rng(3).standard_normal((n, 3))
    X = np.zeros((n, 3))
    st = np.zeros(8, dtype=np.int64)
    rc = hostcheck.hc_amg_solve(C.c_int64(n), _lib.ptr(_lib.i64(A.indptr)), _lib.ptr(_lib.i32(A.indices)),
                                _lib.ptr(np.ascontiguousarray(A.data)), _lib.ptr(B), _lib.ptr(X),
                                C.c_double(1e-10), C.c_int(500), _lib.ptr(st))
    assert rc == 0
    its, levels = int(st[0]), int(st[1])
    ref = spla.spsolve(A.tocsc(), B)
    assert levels >= 2 and st[3] < n / 4  # real coarsening
    assert its <= 60, its
    np.testing.assert_allclose(X, ref, rtol=0, atol=1e-8 * np.abs(ref).max())


def test_torch_ops_registered_and_refuse_cpu_tensors(built_lib):
    import torch
    from paper_1604_07378_b200 import torch_ops  # noqa: F401 (registers the ops)
    for name in ("svd_rv", "material_eval", "factor_solve", "objective", "frame_step"):
        assert hasattr(torch.ops.qnsim_b200, name)
    with pytest.raises(RuntimeError, match="CUDA tensor"):
        torch.ops.qnsim_b200.svd_rv(torch.zeros((2, 3, 3), dtype=torch.float64))
