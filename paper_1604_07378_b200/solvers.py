"""Per-frame quasi-Newton / L-BFGS minimisation on the B200 (mirror of
qnsim.solvers, solvers.py:1-407).

`simulate_frame` keeps the reference signature and return types
(solvers.py:260-352); the whole frame — inertia target, L-BFGS two-loop with
the prefactored A as H0, Armijo backtracking, early-outs, stagnation — runs as
one CUDA-graph launch (`qn_frame_step`).  Every solver kind and L-BFGS
initialisation of solvers.py:25-27 is supported: "pd_qn", "lbfgs" (all three
`lbfgs_init`s) and "chebyshev" run in the device frame graph; "newton" (and
`newton_reference`, the minima for `relative_error`) runs its frame control on
the host like the reference, with per-element Hessian blocks and assembly on
the device and the dense Cholesky by cuSOLVER.  Device-side limits: m <=
QN_MAX_M, alpha_shrink < 1 with a line search (the reference would loop
forever without acceptance), newton without colliders / on single instances.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from paper_1604_07378_b200 import _lib
from paper_1604_07378_b200.dynamics import SimState, SimSystem

SOLVER_KINDS = ("pd_qn", "lbfgs", "chebyshev", "newton")          # solvers.py:25
LBFGS_INITS = ("system_matrix", "scaled_identity", "rest_pose_hessian")
CURVATURE_GUARD = 1e-12
ALPHA_FLOOR = 1e-12


class SolverError(Exception):
    pass


class StagnationError(SolverError):
    """Line search step underflow (solvers.py:39-40)."""


@dataclass
class SolverConfig:
    """solvers.py:43-68 (same defaults and validation)."""

    kind: str = "pd_qn"
    iterations: int = 10
    m: int = 5
    gamma: float = 0.3
    alpha_init: float = 2.0
    alpha_shrink: float = 0.5
    rho: float = 0.9
    S: int = 10
    lbfgs_init: str = "system_matrix"
    line_search: bool = True

    def __post_init__(self):
        if self.kind not in SOLVER_KINDS:
            raise SolverError(f"unknown solver kind {self.kind!r}; valid: {SOLVER_KINDS}")
        if not (0.0 < self.gamma < 1.0):
            raise SolverError(f"gamma must be in (0, 1), got {self.gamma}")
        if self.m < 0:
            raise SolverError("m must be >= 0")
        if not (0.0 <= self.rho < 1.0):
            raise SolverError(f"rho must be in [0, 1), got {self.rho}")
        if self.iterations < 1:
            raise SolverError("iterations must be >= 1")
        if self.lbfgs_init not in LBFGS_INITS:
            raise SolverError(f"unknown lbfgs_init {self.lbfgs_init!r}; valid: {LBFGS_INITS}")

    def to_c(self) -> _lib.SolverConfigC:
        if self.kind not in ("pd_qn", "lbfgs", "chebyshev"):
            raise NotImplementedError(f"solver kind {self.kind!r} is outside the B200 hot path (SURVEY §8f)")

        if self.m > _lib.QN_MAX_M:
            raise NotImplementedError(f"history window m > {_lib.QN_MAX_M}")
        if self.line_search and self.alpha_shrink >= 1.0 and self.alpha_init >= ALPHA_FLOOR:
            # solvers.py:247-252 never reaches the floor: the reference loops until
            # some trial is accepted; the device frame needs a bounded pass count
            raise SolverError(f"alpha_shrink must be < 1 with a line search, got {self.alpha_shrink}")
        c = _lib.SolverConfigC()
        c.kind = {"pd_qn": 0, "lbfgs": 1, "chebyshev": 2}[self.kind]
        c.rho, c.S = float(self.rho), int(self.S)
        c.lbfgs_init = {"system_matrix": 0, "scaled_identity": 1, "rest_pose_hessian": 2}[self.lbfgs_init] \
            if self.kind == "lbfgs" else 0
        c.iterations, c.m, c.line_search = self.iterations, self.m, 1 if self.line_search else 0
        c.gamma, c.alpha_init, c.alpha_shrink = self.gamma, self.alpha_init, self.alpha_shrink
        return c


@dataclass
class ConvergenceRecord:
    """solvers.py:71-80"""

    g0: float = 0.0
    g: list = field(default_factory=list)
    ls_trials: list = field(default_factory=list)
    alphas: list = field(default_factory=list)
    cum_ms: list = field(default_factory=list)
    rel_error: list = field(default_factory=list)
    fallbacks: int = 0
    stagnated: bool = False


def relative_error(g_k: float, g_0: float, g_star: float) -> float:
    """solvers.py:106-110"""
    if g_0 <= g_star + 1e-15:
        raise SolverError(f"degenerate frame: g_0 ({g_0}) not above g* ({g_star})")
    return (g_k - g_star) / (g_0 - g_star)


class _RecordBuffers:
    def __init__(self, n_inst, iterations):
        self.g0 = np.zeros(n_inst)
        self.g = np.zeros((n_inst, iterations))
        self.trials = np.zeros((n_inst, iterations), dtype=np.int32)
        self.alphas = np.zeros((n_inst, iterations))
        self.ms = np.zeros((n_inst, iterations))
        self.status = np.zeros(n_inst, dtype=np.int32)
        self.fallbacks = np.zeros(n_inst, dtype=np.int32)
        self.c = _lib.FrameRecord(_lib.ptr(self.g0), _lib.ptr(self.g), _lib.ptr(self.trials), _lib.ptr(self.alphas),
                                  _lib.ptr(self.ms), _lib.ptr(self.status), _lib.ptr(self.fallbacks))

    def records(self):
        if len(self.g0) > 64:  # batches: build the records without collector pauses
            import gc
            was = gc.isenabled()
            gc.disable()
            try:
                return self._records()
            finally:
                if was:
                    gc.enable()
        return self._records()

    def _records(self):
        g0, g, tr = self.g0.tolist(), self.g.tolist(), self.trials.tolist()
        al, ms, stg = self.alphas.tolist(), self.ms.tolist(), (self.status & 1).astype(bool).tolist()
        fb = self.fallbacks.tolist()
        return [ConvergenceRecord(g0=g0[b], g=g[b], ls_trials=tr[b], alphas=al[b], cum_ms=ms[b], stagnated=stg[b],
                                  fallbacks=fb[b]) for b in range(len(g0))]

    def raise_on_error(self):
        bad = np.nonzero(self.status & 2)[0]
        if bad.size:
            raise SolverError(f"line search requires a descent direction (instance {int(bad[0])})")
        bad = np.nonzero(self.status & 4)[0]
        if bad.size:
            raise SolverError(f"PCG stopped at pcg_maxit before reaching pcg_tol (instance {int(bad[0])})")


NEWTON_FD_STEP_REL = 1e-6   # solvers.py:32
HESSIAN_EIG_FLOOR = 1e-8    # solvers.py:31


def direction_newton(system: SimSystem, state: SimState, x, grad=None) -> np.ndarray:
    """solvers.py:228-234 on the device: central-difference element Hessians,
    eigenvalue floor, dense free-dof Hessian + M/h^2, Cholesky (qn_newton_direction)."""
    from paper_1604_07378_b200.dynamics import gradient
    from paper_1604_07378_b200.linalg import FactorizationError
    if system.colliders:
        raise NotImplementedError("newton with colliders is outside the B200 path")
    if grad is None:
        grad = gradient(system, state, x)
    xs, gs = _lib.f64(x), _lib.f64(grad)
    d = np.empty_like(xs)
    rc = _lib.load().qn_newton_direction(system._h, _lib.ptr(xs), _lib.ptr(gs),
                                         C.c_double(NEWTON_FD_STEP_REL * system.scale),
                                         C.c_double(HESSIAN_EIG_FLOOR), _lib.ptr(d), _lib.QN_MEM_HOST, None)
    if rc == _lib.QN_ERR_NOT_SPD:
        raise FactorizationError(_lib.load().qn_last_error().decode())
    _lib.check(rc, "newton_direction")
    return d


def direction_pd_qn(system: SimSystem, grad) -> np.ndarray:
    """solvers.py:113-117 with the device factor."""
    if system.sysfact is None:
        raise NotImplementedError("pd_qn direction on the host needs a prefactored (direct) system")
    d = np.zeros_like(grad)
    d[system.free] = -system.sysfact.solve(np.ascontiguousarray(grad[system.free]))
    return d


def _line_search(system, st, x, d, g_x, grad, config):
    """solvers.py:241-257"""
    from paper_1604_07378_b200.dynamics import objective
    slope = float(np.vdot(grad, d))
    if slope >= 0.0:
        raise SolverError(f"line search requires a descent direction (slope={slope})")
    alpha, trials = config.alpha_init, 0
    while True:
        alpha *= config.alpha_shrink
        if alpha < 1e-12:
            raise StagnationError("step size underflow")
        trials += 1
        x_new = x + alpha * d
        g_new = objective(system, st, x_new)
        if g_new <= g_x + config.gamma * alpha * slope:
            return alpha, x_new, g_new, trials


def _simulate_frame_newton(system, state, config, fixed_targets):
    """simulate_frame (solvers.py:260-352) for kind="newton": the frame control
    on the host, every objective / gradient / direction on the device."""
    import time
    from paper_1604_07378_b200.dynamics import gradient, inertia_target, objective
    if system.n_inst != 1:
        raise NotImplementedError("newton: single-instance systems")
    t0 = time.perf_counter()
    y = inertia_target(state, system, fixed_targets)
    st = SimState(q_l=state.q_l, q_prev=state.q_prev, y=y)
    x = y.copy()
    rec = ConvergenceRecord()
    grad_tol = 1e-12 * system.scale * max(1.0, float(system.masses.max()) / system.h ** 2)

    def log(g, tr, a):
        rec.g.append(g)
        rec.ls_trials.append(tr)
        rec.alphas.append(a)
        rec.cum_ms.append(1000.0 * (time.perf_counter() - t0))

    rec.g0 = objective(system, st, x)
    for _ in range(config.iterations):
        g_x = objective(system, st, x)
        grad = gradient(system, st, x)
        if float(np.linalg.norm(grad)) <= grad_tol:
            log(g_x, 0, 0.0)
            continue
        d = direction_newton(system, st, x, grad)
        if float(np.vdot(grad, d)) >= 0.0:
            d = direction_pd_qn(system, grad)
            rec.fallbacks += 1
        if config.line_search:
            slope = float(np.vdot(grad, d))
            if slope < 0.0 and -slope <= 1e-12 * max(abs(g_x), 1.0):
                log(g_x, 0, 0.0)
                continue
            try:
                alpha, x_new, g_new, trials = _line_search(system, st, x, d, g_x, grad, config)
            except StagnationError:
                rec.stagnated = True
                while len(rec.g) < config.iterations:
                    log(g_x, 0, 0.0)
                break
        else:
            alpha, x_new, trials = 1.0, x + d, 1
            g_new = objective(system, st, x_new)
        x = x_new
        log(g_new, trials, alpha)
    return SimState(q_l=x, q_prev=np.asarray(state.q_l), y=y), rec


def as_config(config) -> SolverConfig:
    """This package's SolverConfig from any object with the reference's fields
    (qnsim.solvers.SolverConfig, solvers.py:43-68), validated the same way."""
    if config is None or isinstance(config, SolverConfig):
        return config
    return SolverConfig(kind=config.kind, iterations=config.iterations, m=config.m, gamma=config.gamma,
                        alpha_init=config.alpha_init, alpha_shrink=config.alpha_shrink, rho=config.rho, S=config.S,
                        lbfgs_init=config.lbfgs_init, line_search=config.line_search)


def newton_reference(system: SimSystem, state: SimState, fixed_targets=None, grad_tol_rel: float = 1e-10,
                     max_iterations: int = 200, config: SolverConfig | None = None):
    """solvers.py:355-398: the frame solved to (near) optimality with Newton;
    returns (x*, g*), the reference minimum for relative errors."""
    from paper_1604_07378_b200.dynamics import gradient, inertia_target, objective
    config = as_config(config) or SolverConfig(kind="newton", iterations=1)
    y = inertia_target(state, system, fixed_targets)
    st = SimState(q_l=state.q_l, q_prev=state.q_prev, y=y)
    x = y.copy()
    grad0 = gradient(system, st, x)
    tol = grad_tol_rel * max(1.0, float(np.linalg.norm(grad0)))
    g_x = objective(system, st, x)
    best, stalled = np.inf, 0
    for _ in range(max_iterations):
        g_x = objective(system, st, x)
        grad = gradient(system, st, x)
        gn = float(np.linalg.norm(grad))
        if gn <= tol:
            break
        if gn >= 0.999 * best:
            stalled += 1
            if stalled >= 3:
                break
        else:
            stalled = 0
        best = min(best, gn)
        d = direction_newton(system, st, x, grad)
        if float(np.vdot(grad, d)) >= 0.0:
            d = direction_pd_qn(system, grad)
        try:
            _, x, g_x, _ = _line_search(system, st, x, d, g_x, grad, config)
        except StagnationError:
            break
    return x, g_x


def _prepare(system: SimSystem, config: SolverConfig):
    """lbfgs_init="rest_pose_hessian": the rest-pose Hessian is factored (and
    inverted) once per system, lazily (dynamics.py:307, solvers.py:401-407)."""
    if config.kind == "lbfgs" and config.lbfgs_init == "rest_pose_hessian" and \
            not getattr(system, "_rest_hessian_ready", False):
        from paper_1604_07378_b200.linalg import FactorizationError
        rest = _lib.f64(system.mesh.vertices)
        rc = _lib.load().qn_system_rest_hessian(system._h, _lib.ptr(rest),
                                                C.c_double(NEWTON_FD_STEP_REL * system.scale),
                                                C.c_double(HESSIAN_EIG_FLOOR))
        if rc == _lib.QN_ERR_NOT_SPD:
            raise FactorizationError(_lib.load().qn_last_error().decode())
        _lib.check(rc, "rest_pose_hessian")
        system._rest_hessian_ready = True


def simulate_frame(system: SimSystem, state: SimState, config: SolverConfig, fixed_targets=None,
                   out: SimState | None = None):
    """Advance one frame; returns (next_state, ConvergenceRecord) — a list of
    records for batch systems (solvers.py:260-352).  `out` (optional, not in
    the reference signature): a SimState whose q_l / y arrays (float64,
    C-contiguous, e.g. page-locked) receive x and y instead of new arrays.
    `config` may be the reference's own SolverConfig (same fields)."""
    config = as_config(config)
    if config.kind == "newton":
        return _simulate_frame_newton(system, state, config, fixed_targets)
    _prepare(system, config)
    cfg = config.to_c()
    shape = (system.n_inst, system.n, 3) if system.n_inst > 1 else (system.n, 3)
    q_l = _lib.f64(state.q_l).reshape(shape)
    q_prev = _lib.f64(state.q_prev).reshape(shape)
    tg = None
    if fixed_targets is not None and system.fixed.size:
        tg = _lib.f64(np.broadcast_to(fixed_targets, (system.n_inst, system.fixed.size, 3)))
    if out is not None:
        x, y = out.q_l, out.y
        for a in (x, y):
            if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous
                    and a.size == int(np.prod(shape))):
                raise ValueError("simulate_frame: out.q_l / out.y must be C-contiguous float64 of the state's size")
    else:
        x = np.empty(shape)
        y = np.empty(shape)
    rb = _RecordBuffers(system.n_inst, config.iterations)
    rc = _lib.load().qn_simulate_frame(system._h, C.byref(cfg), _lib.ptr(q_l), _lib.ptr(q_prev), _lib.ptr(tg),
                                       _lib.ptr(x), _lib.ptr(y), C.byref(rb.c), _lib.QN_MEM_HOST, None)
    _lib.check(rc, "simulate_frame")
    rb.raise_on_error()
    recs = rb.records()
    nxt = SimState(q_l=x, q_prev=np.asarray(state.q_l), y=y)
    return nxt, (recs[0] if system.n_inst == 1 else recs)


class ResidentRun:
    """Device-resident frame stepping (the state never leaves HBM):
    set_state once, then step() advances q_l/q_prev in place — the `value`
    path of bench.py.  `last_ms` is the CUDA-event time of the last frame."""

    def __init__(self, system: SimSystem, state: SimState, config: SolverConfig):
        config = as_config(config)
        self.system, self.config = system, config
        _prepare(system, config)
        self._cfg = config.to_c()
        shape = (system.n_inst, system.n, 3) if system.n_inst > 1 else (system.n, 3)
        _lib.check(_lib.load().qn_state_set(system._h, _lib.ptr(_lib.f64(state.q_l).reshape(shape)),
                                            _lib.ptr(_lib.f64(state.q_prev).reshape(shape)), _lib.QN_MEM_HOST, None))
        self.shape = shape

    def step(self, fixed_targets=None, record: bool = False, sync: bool = True, stream=None):
        tg = None
        if fixed_targets is not None and self.system.fixed.size:
            tg = _lib.f64(np.broadcast_to(fixed_targets, (self.system.n_inst, self.system.fixed.size, 3)))
        rb = _RecordBuffers(self.system.n_inst, self.config.iterations) if record else None
        _lib.check(_lib.load().qn_frame_step(self.system._h, C.byref(self._cfg), _lib.ptr(tg),
                                             C.byref(rb.c) if rb else None, _lib.QN_MEM_HOST,
                                             1 if (sync or record) else 0, stream), "frame_step")
        if rb:
            rb.raise_on_error()
            return rb.records()
        return None

    def state(self):
        ql = np.empty(self.shape)
        qp = np.empty(self.shape)
        y = np.empty(self.shape)
        _lib.check(_lib.load().qn_state_get(self.system._h, _lib.ptr(ql), _lib.ptr(qp), _lib.ptr(y),
                                            _lib.QN_MEM_HOST, None))
        return SimState(q_l=ql, q_prev=qp, y=y)

    @property
    def last_ms(self) -> float:
        v = C.c_double(0.0)
        _lib.check(_lib.load().qn_system_last_frame_ms(self.system._h, C.byref(v)))
        return v.value

    @property
    def last_passes(self) -> int:
        v = C.c_int64(0)
        _lib.check(_lib.load().qn_system_last_frame_passes(self.system._h, C.byref(v)))
        return v.value

    @property
    def last_cg_iterations(self) -> int:
        v = C.c_int64(0)
        _lib.check(_lib.load().qn_system_last_frame_cg_iterations(self.system._h, C.byref(v)))
        return v.value
