"""PyTorch custom ops over the C-ABI (the thin boundary BASELINE.json's
north_star asks for): device tensors in, device tensors out, on the current
torch stream, no host round trip.  Each op is one call into
libqnsim_b200.so with QN_MEM_DEVICE pointers; there is no CPU implementation
(a CPU tensor raises), so a torch program that uses these ops always runs
the sm_100a kernels.

    torch.ops.qnsim_b200.svd_rv(F)                    # (m,3,3) -> U, sigma, V   (linalg.py:86-110)
    torch.ops.qnsim_b200.material_eval(h, sigma)      # (k,3)   -> psi, tau      (materials.py:184-197)
    torch.ops.qnsim_b200.factor_solve(h, B, batch)    # (n,3)   -> A^-1 B        (linalg.py:36-40)
    torch.ops.qnsim_b200.objective(h, x, y)           # (n,3)   -> g, grad       (dynamics.py:460-478)
    torch.ops.qnsim_b200.frame_step(h, n_inst, its, m, kind)  # resident frame -> g, status (solvers.py:260-352)

`h` is an integer handle: `register_material(mat)`, `Factorization.op_handle`
or `SimSystem.op_handle`.
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _lib

_MATERIALS: dict[int, object] = {}  # handle -> ctypes qn_material (kept alive)


def _dev(t: torch.Tensor, name: str) -> torch.Tensor:
    if not t.is_cuda:
        raise RuntimeError(f"qnsim_b200: {name} must be a CUDA tensor (no CPU implementation)")
    return t.contiguous().to(torch.float64)


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def register_material(material) -> int:
    """Handle of a material descriptor for `material_eval` (MaterialModel or builtin)."""
    c = material.to_c()
    h = C.addressof(c)
    _MATERIALS[h] = c
    return h


@torch.library.custom_op("qnsim_b200::svd_rv", mutates_args=())
def svd_rv(F: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    F = _dev(F, "F")
    m = F.shape[0]
    U = torch.empty_like(F)
    V = torch.empty_like(F)
    s = torch.empty((m, 3), dtype=torch.float64, device=F.device)
    _lib.check(_lib.load().qn_svd_rv_batch(C.c_int64(m), C.c_void_p(F.data_ptr()), C.c_void_p(U.data_ptr()),
                                           C.c_void_p(s.data_ptr()), C.c_void_p(V.data_ptr()), _lib.QN_MEM_DEVICE,
                                           C.c_void_p(_stream())), "svd_rv")
    return U, s, V


@svd_rv.register_fake
def _(F):
    return torch.empty_like(F), F.new_empty((F.shape[0], 3)), torch.empty_like(F)


@torch.library.custom_op("qnsim_b200::material_eval", mutates_args=())
def material_eval(handle: int, sigma: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    sigma = _dev(sigma, "sigma")
    k = sigma.shape[0]
    psi = torch.empty((k,), dtype=torch.float64, device=sigma.device)
    tau = torch.empty_like(sigma)
    _lib.check(_lib.load().qn_material_eval(C.c_void_p(handle), C.c_int64(k), C.c_void_p(sigma.data_ptr()),
                                            C.c_void_p(psi.data_ptr()), C.c_void_p(tau.data_ptr()),
                                            _lib.QN_MEM_DEVICE, C.c_void_p(_stream())), "material_eval")
    return psi, tau


@material_eval.register_fake
def _(handle, sigma):
    return sigma.new_empty((sigma.shape[0],)), torch.empty_like(sigma)


@torch.library.custom_op("qnsim_b200::factor_solve", mutates_args=())
def factor_solve(handle: int, B: torch.Tensor, batch: int) -> torch.Tensor:
    B = _dev(B, "B")
    X = torch.empty_like(B)
    _lib.check(_lib.load().qn_factor_solve(C.c_void_p(handle), C.c_int64(batch), C.c_void_p(B.data_ptr()),
                                           C.c_void_p(X.data_ptr()), C.c_int64(B.shape[1] if B.dim() > 1 else 1),
                                           _lib.QN_MEM_DEVICE, C.c_void_p(_stream())), "factor_solve")
    return X


@factor_solve.register_fake
def _(handle, B, batch):
    return torch.empty_like(B)


@torch.library.custom_op("qnsim_b200::objective", mutates_args=())
def objective(handle: int, x: torch.Tensor, y: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """g (one per instance) and the gradient with fixed rows zeroed, at x."""
    x, y = _dev(x, "x"), _dev(y, "y")
    n_inst = x.shape[0] if x.dim() == 3 else 1
    g = torch.empty((n_inst,), dtype=torch.float64, device=x.device)
    grad = torch.empty_like(x)
    _lib.check(_lib.load().qn_system_objective(C.c_void_p(handle), C.c_void_p(x.data_ptr()),
                                               C.c_void_p(y.data_ptr()), C.c_void_p(g.data_ptr()),
                                               C.c_void_p(grad.data_ptr()), _lib.QN_MEM_DEVICE,
                                               C.c_void_p(_stream())), "objective")
    return g, grad


@objective.register_fake
def _(handle, x, y):
    return x.new_empty((x.shape[0] if x.dim() == 3 else 1,)), torch.empty_like(x)


@torch.library.custom_op("qnsim_b200::frame_step", mutates_args=())
def frame_step(handle: int, n_inst: int, iterations: int, m: int, kind: int) -> tuple[torch.Tensor, torch.Tensor]:
    """One frame on the resident state of system `handle` (state set with
    qn_state_set / ResidentRun; kind 1 = lbfgs, 0 = pd_qn), enqueued on the
    current stream with no host synchronisation.  Returns the per-iteration
    objective g of every instance, (n_inst, iterations), and the per-instance
    status (bit 0 stagnated, bit 1 ascent = the reference's SolverError), both
    device tensors written by the device (qn_frame_records_device)."""
    from .solvers import SolverConfig
    cfg = SolverConfig(kind="lbfgs" if kind == 1 else "pd_qn", iterations=iterations, m=m).to_c()
    dev = torch.device("cuda", torch.cuda.current_device())
    g = torch.empty((n_inst, iterations), dtype=torch.float64, device=dev)
    status = torch.empty((n_inst,), dtype=torch.int32, device=dev)
    lib = _lib.load()
    _lib.check(lib.qn_frame_step(C.c_void_p(handle), C.byref(cfg), None, None, _lib.QN_MEM_DEVICE, 0,
                                 C.c_void_p(_stream())), "frame_step")
    _lib.check(lib.qn_frame_records_device(C.c_void_p(handle), iterations, C.c_void_p(g.data_ptr()),
                                           C.c_void_p(status.data_ptr()), C.c_void_p(_stream())), "frame_step")
    return g, status


@frame_step.register_fake
def _(handle, n_inst, iterations, m, kind):
    return (torch.empty((n_inst, iterations), dtype=torch.float64, device="cuda"),
            torch.empty((n_inst,), dtype=torch.int32, device="cuda"))
