"""Python mirror of the reference's projection / optimizer-step interface.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/topt/projection.hpp:17-109 and errors.hpp:9-42
(and SPEC.md:272-313 for the optimizer step, which has no reference code), so
parity tests read like the reference's own tests.  Every function runs on the
GPU through the C-ABI (include/topt_b200.h); there is no CPU path.

Host numpy arrays use the host-buffer entry points (H2D/D2H inside the
call); torch CUDA tensors use the *_dev entry points (no copies).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
from typing import Optional, Sequence

import numpy as np

from . import _lib as L


# ---- errors.hpp:9-42 ---------------------------------------------------------
class ParameterError(ValueError):
    """topt::ParameterError (std::invalid_argument)."""


class DomainError(ValueError):
    """topt::DomainError (std::domain_error)."""


class SingularSystemError(RuntimeError):
    """topt::SingularSystemError."""


class InfeasibleLinearization(RuntimeError):
    """topt::InfeasibleLinearization."""


class NumericalError(RuntimeError):
    """topt::NumericalError."""


class UnsupportedProblem(RuntimeError):
    """topt::UnsupportedProblem."""


class CudaError(RuntimeError):
    """CUDA runtime failure inside the library."""


_ERRMAP = {L.ERR_PARAMETER: ParameterError, L.ERR_DOMAIN: DomainError,
           L.ERR_SINGULAR: SingularSystemError, L.ERR_INFEASIBLE: InfeasibleLinearization,
           L.ERR_NUMERICAL: NumericalError, L.ERR_UNSUPPORTED: UnsupportedProblem,
           L.ERR_CUDA: CudaError, L.ERR_INTERNAL: RuntimeError}


def _check(ctx: L.Context, rc: int):
    if rc != L.OK:
        raise _ERRMAP.get(rc, RuntimeError)(ctx.last_error())


# ---- projection.hpp:43-64 ----------------------------------------------------
class ProjectionPath(enum.IntEnum):
    single_binary = 0
    independent_binary = 1
    newton = 2


def to_string(path) -> str:
    try:
        return ProjectionPath(int(path)).name
    except ValueError:
        return "unknown"


@dataclasses.dataclass
class ProjectionOptions:
    c: float = 1e12
    tol_b: float = 1e-8
    tol_n: float = 1e-6
    newton_maxiter: int = 50
    binary_maxiter: int = 200

    def _c(self):
        return L.ProjOptions(self.c, self.tol_b, self.tol_n, self.newton_maxiter,
                             self.binary_maxiter)


@dataclasses.dataclass
class ProjectionResult:
    delta: object
    y: np.ndarray
    slacks: np.ndarray
    path: ProjectionPath = ProjectionPath.single_binary
    newton_iters: int = 0
    residual: float = 0.0
    converged: bool = True
    curvature_violations: int = 0
    # diagnostics (not in the reference)
    passes: int = 0
    sweeps: int = 0
    stage1_row: int = -1
    near_ties: int = 0
    min_margin: float = float("inf")
    bisect_iters: Optional[list] = None
    mask: object = None
    local_sweeps: int = 0
    gathered: bool = False
    exact_passes: int = 0


class parity:
    """Context manager: run the enclosed calls on `device` in the given parity
    mode ('strict' or 'certified'; include/topt_b200.h), restoring the old one."""

    def __init__(self, mode: str, device: int = 0):
        self.mode, self.device = mode, device

    def __enter__(self):
        self.ctx = L.context(self.device)
        self.old = self.ctx.parity
        self.ctx.set_parity(self.mode)
        return self.ctx

    def __exit__(self, *a):
        self.ctx.set_parity(self.old)
        return False


def _meta_to_result(meta: L.ProjMeta, delta, y, slacks, m, mask=None) -> ProjectionResult:
    return ProjectionResult(
        delta=delta, y=y, slacks=slacks, path=ProjectionPath(meta.path),
        newton_iters=meta.newton_iters, residual=meta.residual,
        converged=bool(meta.converged), curvature_violations=meta.curvature_violations,
        passes=meta.passes, sweeps=meta.sweeps, stage1_row=meta.stage1_row,
        near_ties=meta.near_ties, min_margin=meta.min_margin,
        bisect_iters=list(meta.bisect_iters[:m]), mask=mask, local_sweeps=meta.local_sweeps,
        gathered=bool(meta.gathered), exact_passes=meta.exact_passes)


def _is_torch_cuda(a) -> bool:
    return hasattr(a, "is_cuda") and bool(a.is_cuda)


def _ptr(a):
    if a is None:
        return None
    if _is_torch_cuda(a):
        return a.data_ptr()
    return a.ctypes.data


def _dev_f64(a, name, numel=None, device=None):
    """A torch CUDA tensor the C-ABI may read as contiguous fp64 at data_ptr():
    float64, on `device` (a torch.device or None), `numel` elements; strided
    views are made contiguous (the caller keeps the returned tensor alive).
    Anything else is a DomainError -- never silently reinterpreted."""
    import torch
    if a.dtype != torch.float64:
        raise DomainError(f"{name}: expected a float64 tensor, got {a.dtype}")
    if device is not None and a.device != device:
        raise DomainError(f"{name}: tensor on {a.device}, expected {device}")
    if numel is not None and a.numel() != numel:
        raise DomainError(f"{name}: {a.numel()} elements, expected {numel}")
    return a if a.is_contiguous() else a.contiguous()


def _f64(a, name="array"):
    if a is None:
        return a
    if _is_torch_cuda(a):
        return _dev_f64(a, name)
    return np.ascontiguousarray(a, dtype=np.float64)


def _part_csr(partition, m):
    if partition is None:
        return None, None
    if len(partition) != m:
        raise DomainError("ConstraintLinearization: partition size != m")
    off = np.zeros(m + 1, np.int64)
    for j, p in enumerate(partition):
        off[j + 1] = off[j] + len(p)
    idx = (np.concatenate([np.asarray(p, dtype=np.int32).ravel() for p in partition])
           if m else np.zeros(0, np.int32))
    return off, np.ascontiguousarray(idx, dtype=np.int32)


# ---- ConstraintLinearization (projection.hpp:17-41) --------------------------
class ConstraintLinearization:
    """Per-iteration linearization; g_hat is computed on the GPU by build()."""

    def __init__(self):
        self.num_constraints = 0
        self.num_vars = 0
        self.grad = None
        self.g_values = None
        self.bounds_g = None
        self.gd_step = None
        self.g_hat = None
        self.g_hat_err = None
        self.is_equality = None
        self.partition = None
        self._device = 0
        self._owner = None

    @staticmethod
    def build(m, n, grad, g_values, bounds_g, gd_step, is_equality=None, partition=None,
              device: int = 0) -> "ConstraintLinearization":
        lin = ConstraintLinearization()
        lin.num_constraints = int(m)
        lin.num_vars = int(n)
        lin._device = device
        if _is_torch_cuda(grad):
            grad = _dev_f64(grad, "grad", m * n)
            lin.grad = grad.reshape(m, n) if m * n else grad
        else:
            lin.grad = np.ascontiguousarray(np.asarray(grad, np.float64).reshape(-1))
        lin.g_values = np.ascontiguousarray(g_values, np.float64).reshape(-1)
        lin.bounds_g = np.ascontiguousarray(bounds_g, np.float64).reshape(-1)
        lin.gd_step = _f64(gd_step, "gd_step")
        lin.is_equality = (np.zeros(m, np.uint8) if is_equality is None or len(is_equality) == 0
                           else np.ascontiguousarray(is_equality, np.uint8))
        lin.partition = partition
        gsz = lin.grad.numel() if _is_torch_cuda(lin.grad) else lin.grad.size
        gdsz = lin.gd_step.numel() if _is_torch_cuda(lin.gd_step) else np.asarray(lin.gd_step).size
        if (gsz != m * n or lin.g_values.size != m or lin.bounds_g.size != m or gdsz != n
                or lin.is_equality.size != m):
            raise DomainError("ConstraintLinearization: inconsistent dimensions")
        if not _is_torch_cuda(lin.grad):
            lin.grad = lin.grad.reshape(m, n)
        ctx = L.context(device)
        g_hat = np.zeros(m)
        g_err = np.zeros(m)
        with _LinC(lin, need_gd=True) as lc:
            if lc.device_mode:
                raise DomainError("build() takes host arrays; use pgd_step_device for device data")
            _check(ctx, ctx.lib.topt_b200_build(ctx.h, C.byref(lc.s), _ptr(g_hat), _ptr(g_err)))
        lin.g_hat = g_hat
        lin.g_hat_err = g_err
        return lin

    def row(self, j):
        return self.grad[j]

    def validate(self):
        """Recheck g_hat (1e-14) and partition validity (projection.cpp:150-181)."""
        m = self.num_constraints
        if self.partition is not None and len(self.partition) != m:
            raise DomainError("ConstraintLinearization: partition size != m")
        fresh = ConstraintLinearization.build(m, self.num_vars, self.grad, self.g_values,
                                              self.bounds_g, self.gd_step, self.is_equality,
                                              self.partition, self._device)
        for j in range(m):
            expect = fresh.g_hat[j]
            scale = max(1.0, abs(expect), abs(self.g_hat[j]))
            if abs(self.g_hat[j] - expect) > 1e-14 * scale + self.g_hat_err[j]:
                raise DomainError("ConstraintLinearization: g_hat inconsistent with fields")


class _LinC:
    """Builds the C topt_linearization view (keeps buffers alive)."""

    def __init__(self, lin: ConstraintLinearization, need_gd=False, ghat=True):
        self.lin = lin
        self.need_gd = need_gd
        self.ghat = ghat

    def __enter__(self):
        lin = self.lin
        m = lin.num_constraints
        self.device_mode = _is_torch_cuda(lin.grad)
        self.off, self.idx = _part_csr(lin.partition, m)
        s = L.Linearization()
        s.num_constraints = m
        s.num_vars = lin.num_vars
        s.grad = _ptr(lin.grad)
        s.g_values = _ptr(lin.g_values)
        s.bounds_g = _ptr(lin.bounds_g)
        s.gd_step = _ptr(lin.gd_step) if (self.need_gd and lin.gd_step is not None) else None
        self._gh = None if lin.g_hat is None else np.ascontiguousarray(lin.g_hat, np.float64)
        self._ge = None if lin.g_hat_err is None else np.ascontiguousarray(lin.g_hat_err,
                                                                          np.float64)
        s.g_hat = _ptr(self._gh)
        s.g_hat_err = _ptr(self._ge)
        s.is_equality = _ptr(lin.is_equality)
        s.part_offsets = _ptr(self.off)
        s.part_indices = _ptr(self.idx)
        s.owner = None
        self.s = s
        return self

    def __exit__(self, *a):
        return False


def _host_only(lin, rho, fn):
    if _is_torch_cuda(rho) or _is_torch_cuda(lin.grad) or _is_torch_cuda(lin.gd_step):
        raise DomainError(f"{fn}: takes host (numpy) arrays")


def _check_rho(lin, rho):
    n = rho.numel() if _is_torch_cuda(rho) else np.asarray(rho).size
    if n != lin.num_vars:
        raise DomainError("projection: rho_tilde size does not match linearization")


# ---- projection.hpp:66-109 ---------------------------------------------------
def delta_of_y(y, lin: ConstraintLinearization, rho_tilde, lower, upper):
    rho = _f64(rho_tilde)
    _host_only(lin, rho, "delta_of_y")
    _check_rho(lin, rho)
    y = np.ascontiguousarray(y, np.float64)
    if y.size != lin.num_constraints:
        raise DomainError("delta_of_y: dual size does not match linearization")
    ctx = L.context(lin._device)
    out = np.empty(lin.num_vars)
    with _LinC(lin) as lc:
        _check(ctx, ctx.lib.topt_b200_delta_of_y(ctx.h, _ptr(y), C.byref(lc.s), _ptr(rho),
                                                 C.c_double(lower), C.c_double(upper),
                                                 _ptr(out)))
    return out


def constraint_residual_h(y, lin: ConstraintLinearization, rho_tilde, lower, upper, c):
    rho = _f64(rho_tilde)
    y = np.ascontiguousarray(y, np.float64)
    if not (c > 0.0):
        raise ParameterError("constraint_residual_h: c must be > 0")
    _host_only(lin, rho, "constraint_residual_h")
    _check_rho(lin, rho)
    if y.size != lin.num_constraints:
        raise DomainError("delta_of_y: dual size does not match linearization")
    ctx = L.context(lin._device)
    out = np.empty(lin.num_constraints)
    with _LinC(lin) as lc:
        _check(ctx, ctx.lib.topt_b200_constraint_residual_h(
            ctx.h, _ptr(y), C.byref(lc.s), _ptr(rho), C.c_double(lower), C.c_double(upper),
            C.c_double(c), _ptr(out)))
    return out


def _project(which, rho_tilde, lin, lower, upper, options: ProjectionOptions,
             want_mask=False):
    rho = _f64(rho_tilde, "rho_tilde")
    if _is_torch_cuda(rho) != _is_torch_cuda(lin.grad):
        raise DomainError("projection: rho_tilde and the linearization must both be host "
                          "arrays or both CUDA tensors")
    if _is_torch_cuda(rho) and lin.grad.device != rho.device:
        raise DomainError("projection: rho_tilde and grad are on different devices")
    _check_rho(lin, rho)
    ctx = L.context(lin._device)
    m, n = lin.num_constraints, lin.num_vars
    y = np.zeros(m)
    sl = np.zeros(m)
    meta = L.ProjMeta()
    opts = options._c()
    with _LinC(lin, need_gd=lin.partition is not None) as lc:
        if lc.device_mode:
            import torch
            delta = torch.empty(n, dtype=torch.float64, device=rho.device)
            mask = torch.empty(n, dtype=torch.uint8, device=rho.device) if want_mask else None
            if lin._owner is None and lin.partition is not None and m > 1:
                lin._owner = torch.empty(n, dtype=torch.int8, device=rho.device)
                _check(ctx, ctx.lib.topt_b200_owner_map(ctx.h, C.c_int64(n), C.c_int32(m),
                                                        _ptr(lc.off), _ptr(lc.idx),
                                                        C.c_void_p(lin._owner.data_ptr())))
            lc.s.owner = None if lin._owner is None else lin._owner.data_ptr()
            with ctx.ordered_with_torch():
                _check(ctx, ctx.lib.topt_b200_project_dev(
                    ctx.h, which, rho.data_ptr(), C.byref(lc.s), lower, upper, C.byref(opts),
                    delta.data_ptr(), mask.data_ptr() if mask is not None else None, _ptr(y),
                    _ptr(sl), C.byref(meta)))
            return _meta_to_result(meta, delta, y, sl, m, mask)
        delta = np.empty(n)
        _check(ctx, ctx.lib.topt_b200_project(ctx.h, which, _ptr(rho), C.byref(lc.s),
                                              C.c_double(lower), C.c_double(upper),
                                              C.byref(opts), _ptr(delta), _ptr(y), _ptr(sl),
                                              C.byref(meta)))
    return _meta_to_result(meta, delta, y, sl, m)


def project_single_binary_search(rho_tilde, lin, lower, upper, tol_b, binary_maxiter=200):
    o = ProjectionOptions(tol_b=tol_b, binary_maxiter=binary_maxiter)
    return _project(L.PROJECT_SINGLE, rho_tilde, lin, lower, upper, o)


def project_independent(rho_tilde, lin, lower, upper, tol_b, binary_maxiter=200):
    o = ProjectionOptions(tol_b=tol_b, binary_maxiter=binary_maxiter)
    return _project(L.PROJECT_INDEPENDENT, rho_tilde, lin, lower, upper, o)


def project_general_newton(rho_tilde, lin, lower, upper, options: ProjectionOptions = None):
    return _project(L.PROJECT_NEWTON, rho_tilde, lin, lower, upper,
                    options or ProjectionOptions())


def project(rho_tilde, lin, lower, upper, options: ProjectionOptions = None, want_mask=False):
    return _project(L.PROJECT_AUTO, rho_tilde, lin, lower, upper,
                    options or ProjectionOptions(), want_mask)


# ---- optimizer step ----------------------------------------
@dataclasses.dataclass
class PgdSettings:
    alpha_max: float = 1e2
    alpha_fallback: float = 0.2
    t_warmup: int = 50
    omega: float = 1.0
    eps_alpha: float = 1e-6
    tol: float = 0.0
    K_max: int = 300
    C: float = 1e12
    tol_B: float = 1e-8
    tol_N: float = 1e-6

    def _c(self):
        return L.PgdSettingsC(self.alpha_max, self.alpha_fallback, self.omega, self.eps_alpha,
                              self.tol_N, self.t_warmup)

    def options(self) -> ProjectionOptions:
        return ProjectionOptions(c=self.C, tol_b=self.tol_B, tol_n=self.tol_N)


@dataclasses.dataclass
class StepResult:
    x_new: object
    d: object
    rho_tilde: object
    delta: object
    y: np.ndarray
    slacks: np.ndarray
    g_hat: np.ndarray
    alpha: float
    beta: float
    fallback: bool
    projection: ProjectionResult
    mask: object = None


class PreparedStep:
    """A PGD step bound to its buffers: the C-ABI call with every argument
    struct built once, so repeated steps on the same buffers (an optimizer
    loop, the benchmark) pay only the library call.  `run()` executes the
    step; `result()` wraps the last outputs like pgd_step's return value."""

    def __init__(self, ctx, fn, args, keep, m, outs, rows=None, dev=False):
        self.ctx, self._fn, self._args, self._keep, self.m = ctx, fn, args, keep, m
        self._outs = outs
        self._rows = rows   # (RowDesc list, grid, index_offset) or None
        self._dev = dev     # device tensors: order the call with torch's stream

    def run(self):
        if self._rows is not None:
            self.ctx.set_structured_rows(*self._rows)
        try:
            if self._dev:
                with self.ctx.ordered_with_torch():
                    _check(self.ctx, self._fn(*self._args))
            else:
                _check(self.ctx, self._fn(*self._args))
        finally:
            if self._rows is not None:
                self.ctx.set_structured_rows(None)
        return self

    def result(self) -> StepResult:
        o = self._outs
        meta = o["meta"]
        proj = _meta_to_result(meta, o["delta"], o["y"].copy(), o["sl"].copy(), self.m, o["mask"])
        return StepResult(x_new=o["x_new"], d=o["d"], rho_tilde=o["rt"], delta=o["delta"],
                          y=o["y"].copy(), slacks=o["sl"].copy(), g_hat=o["gh"].copy(),
                          alpha=meta.alpha,
                          beta=meta.beta, fallback=bool(meta.fallback), projection=proj,
                          mask=o["mask"])


def pgd_step(x, x_prev, g, g_prev, d_prev, grad, g_values, bounds_g, is_equality=None,
             partition=None, t=1, violation=0.0, lower=0.0, upper=1.0,
             settings: PgdSettings = None, device: int = 0, want_delta=False,
             want_mask=False, out=None,
             host_outputs=("x_new", "d", "rho_tilde"), ctx: L.Context = None,
             n_global: int = None, row_counts=None) -> StepResult:
    """One PGD-TO step (Alg. 3 lines 2-15): BB step, PR+ direction, rho_tilde,
    linearization, projection, rho_{t+1} = rho_tilde + delta.

    numpy inputs -> host-buffer C-ABI (copies inside the call);
    torch CUDA tensors -> device C-ABI (no copies; `out` may supply buffers).
    """
    return prepare_pgd_step(x, x_prev, g, g_prev, d_prev, grad, g_values, bounds_g,
                            is_equality, partition, t, violation, lower, upper, settings,
                            device, want_delta, want_mask, out, host_outputs, ctx, n_global,
                            row_counts).run().result()


def prepare_pgd_step(x, x_prev, g, g_prev, d_prev, grad, g_values, bounds_g, is_equality=None,
                     partition=None, t=1, violation=0.0, lower=0.0, upper=1.0,
                     settings: PgdSettings = None, device: int = 0, want_delta=False,
                     want_mask=False, out=None,
                     host_outputs=("x_new", "d", "rho_tilde"), ctx: L.Context = None,
                     n_global: int = None, row_counts=None, rows=None, grid=None,
                     index_offset: int = 0) -> PreparedStep:
    """pgd_step's argument handling without the call: returns a PreparedStep
    whose run() executes the step on these buffers (the arrays are referenced,
    not copied, so updating them in place between runs is allowed).

    rows / grid / index_offset (device tensors only): structured constraint
    rows (a list of dicts {kind: "dense"|"const"|"centroid", value, axis,
    center, scale, sign}); generated rows are never read from `grad`, which
    may then be None."""
    settings = settings or PgdSettings()
    ctx = ctx or L.context(device)
    dev = _is_torch_cuda(x)
    n = int(x.numel() if dev else np.asarray(x).size)
    m = int(len(g_values))
    gv = np.ascontiguousarray(g_values, np.float64)
    bg = np.ascontiguousarray(bounds_g, np.float64)
    ie = None if is_equality is None else np.ascontiguousarray(is_equality, np.uint8)
    off, idx = _part_csr(partition, m)
    pr = L.StepProblem()
    pr.n, pr.m, pr.t, pr.violation, pr.lower, pr.upper = n, m, int(t), float(violation), \
        float(lower), float(upper)
    y = np.zeros(m)
    sl = np.zeros(m)
    gh = np.zeros(m)
    meta = L.ProjMeta()
    opts = settings.options()._c()
    sc = settings._c()
    o = L.StepOutputs()
    o.y, o.slacks, o.g_hat = _ptr(y), _ptr(sl), _ptr(gh)
    if dev:
        import torch
        dv = x.device
        x = _dev_f64(x, "x", n, dv)
        x_prev = _dev_f64(x_prev, "x_prev", n, dv)
        g = _dev_f64(g, "g", n, dv)
        g_prev = _dev_f64(g_prev, "g_prev", n, dv)
        d_prev = _dev_f64(d_prev, "d_prev", n, dv)
        if grad is not None:
            grad = _dev_f64(grad, "grad", m * n, dv)
        elif rows is None:
            raise DomainError("pgd_step: grad is required unless structured rows are given")
        bufs = out or {}
        for k in ("x_new", "d", "rho_tilde", "delta"):
            b = bufs.get(k)
            if b is not None and (b.dtype != torch.float64 or b.device != dv
                                  or b.numel() != n or not b.is_contiguous()):
                raise DomainError(f"pgd_step: out[{k!r}] must be a contiguous float64 tensor "
                                  f"of {n} elements on {dv}")
        x_new = bufs.get("x_new") if bufs.get("x_new") is not None else torch.empty_like(x)
        d = bufs.get("d") if bufs.get("d") is not None else torch.empty_like(x)
        rt = bufs.get("rho_tilde") if bufs.get("rho_tilde") is not None else torch.empty_like(x)
        delta = (bufs.get("delta") if bufs.get("delta") is not None else torch.empty_like(x)) \
            if want_delta else None
        mask = torch.empty(n, dtype=torch.uint8, device=x.device) if want_mask else None
        owner = bufs.get("owner")
        if owner is None and partition is not None and m > 1:
            owner = torch.empty(n, dtype=torch.int8, device=x.device)
            _check(ctx, ctx.lib.topt_b200_owner_map(ctx.h, C.c_int64(n), C.c_int32(m), _ptr(off),
                                                    _ptr(idx), C.c_void_p(owner.data_ptr())))
        for f, a in (("x", x), ("x_prev", x_prev), ("g", g), ("g_prev", g_prev),
                     ("d_prev", d_prev), ("grad", grad)):
            setattr(pr, f, a.data_ptr() if a is not None else None)
        pr.g_values, pr.bounds_g = _ptr(gv), _ptr(bg)
        pr.is_equality = _ptr(ie)
        pr.part_offsets, pr.part_indices = _ptr(off), _ptr(idx)
        pr.owner = owner.data_ptr() if owner is not None else None
        o.x_new, o.d, o.rho_tilde = x_new.data_ptr(), d.data_ptr(), rt.data_ptr()
        o.delta = delta.data_ptr() if delta is not None else None
        o.mask = mask.data_ptr() if mask is not None else None
        if getattr(ctx, "distributed", False):
            rc_arr = None if row_counts is None else np.ascontiguousarray(row_counts, np.int64)
            fn = ctx.lib.topt_b200_pgd_step_ranks
            args = (ctx.h, C.byref(pr), int(n_global if n_global is not None else n),
                    _ptr(rc_arr), C.byref(sc), C.byref(opts), C.byref(o), C.byref(meta))
            keep = [rc_arr]
        else:
            fn = ctx.lib.topt_b200_pgd_step_dev
            args = (ctx.h, C.byref(pr), C.byref(sc), C.byref(opts), C.byref(o), C.byref(meta))
            keep = []
        keep += [x, x_prev, g, g_prev, d_prev, grad, owner]
    else:
        arrs = {k: np.ascontiguousarray(v, np.float64) for k, v in
                (("x", x), ("x_prev", x_prev), ("g", g), ("g_prev", g_prev), ("d_prev", d_prev),
                 ("grad", grad))}
        for f, a in arrs.items():
            setattr(pr, f, a.ctypes.data)
        pr.g_values, pr.bounds_g = _ptr(gv), _ptr(bg)
        pr.is_equality = _ptr(ie)
        pr.part_offsets, pr.part_indices = _ptr(off), _ptr(idx)
        hb = out or {}
        x_new = (hb["x_new"] if hb.get("x_new") is not None else np.empty(n)) \
            if "x_new" in host_outputs else None
        d = (hb["d"] if hb.get("d") is not None else np.empty(n)) \
            if "d" in host_outputs else None
        rt = (hb["rho_tilde"] if hb.get("rho_tilde") is not None else np.empty(n)) \
            if "rho_tilde" in host_outputs else None
        delta = np.empty(n) if want_delta else None
        mask = np.empty(n, np.uint8) if want_mask else None
        o.x_new, o.d, o.rho_tilde = _ptr(x_new), _ptr(d), _ptr(rt)
        o.delta = _ptr(delta)
        o.mask = _ptr(mask)
        fn = ctx.lib.topt_b200_pgd_step
        args = (ctx.h, C.byref(pr), C.byref(sc), C.byref(opts), C.byref(o), C.byref(meta))
        keep = [arrs]
    keep += [pr, sc, opts, o, meta, gv, bg, ie, off, idx]
    outs = dict(meta=meta, delta=delta, y=y, sl=sl, gh=gh, mask=mask, x_new=x_new, d=d, rt=rt)
    srows = None
    if rows is not None:
        if not dev:
            raise ValueError("structured rows need device (torch CUDA) inputs")
        kinds = {"dense": 0, "const": 1, "centroid": 2}
        descs = [L.RowDesc(kinds[r["kind"]], int(r.get("axis", 0)), float(r.get("value", 0.0)),
                           float(r.get("center", 0.0)), float(r.get("scale", 1.0)),
                           float(r.get("sign", 1.0))) for r in rows]
        srows = (descs, grid, index_offset)
    return PreparedStep(ctx, fn, args, keep, m, outs, srows, dev)



# ---- upstream of the step: filter, SIMP, sensitivities ------
@dataclasses.dataclass
class StructuredGrid:
    """grid.hpp:13-21: nx x ny unit-size (or element_size) square elements,
    element e = ey * nx + ex."""
    nx: int = 1
    ny: int = 1
    element_size: float = 1.0

    def __post_init__(self):
        if self.nx < 1 or self.ny < 1:
            raise ParameterError("grid: nx and ny must be >= 1")
        if not (self.element_size > 0.0):
            raise ParameterError("grid: element_size must be > 0")

    def num_elements(self) -> int:
        return self.nx * self.ny

    def num_dofs(self) -> int:
        return 2 * (self.nx + 1) * (self.ny + 1)

    def element_index(self, ex, ey) -> int:
        return ey * self.nx + ex


class FilterKernel:
    """filter.hpp:15-25: the row-normalized hat kernel.  The CSR arrays are the
    reference's (row_ptr, col, weight); the product runs matrix-free on the
    GPU from (nx, ny, radius) when the kernel came from build_filter, and as
    a CSR product otherwise -- both in the reference's summation orders."""

    def __init__(self, size, radius, row_ptr, col, weight, grid=None, handle=None, ctx=None):
        self.size, self.radius = int(size), float(radius)
        self.row_ptr, self.col, self.weight = row_ptr, col, weight
        self._grid, self._h, self._ctx = grid, handle, ctx

    def is_identity(self) -> bool:
        return len(self.col) == self.size

    def __del__(self):
        try:
            if self._h:
                self._ctx.lib.topt_b200_filter_destroy(self._h)
                self._h = None
        except Exception:
            pass


def build_filter(grid: StructuredGrid, radius: float, device: int = 0) -> FilterKernel:
    """build_filter (filter.cpp:10-43)."""
    if not (radius > 0.0):
        raise ParameterError("build_filter: radius must be > 0")
    ctx = L.context(device)
    h = C.c_void_p()
    _check(ctx, ctx.lib.topt_b200_filter_create(ctx.h, grid.nx, grid.ny, float(radius),
                                                C.byref(h)))
    n = grid.num_elements()
    nnz = int(ctx.lib.topt_b200_filter_nnz(h))
    rp = np.empty(n + 1, np.int32); col = np.empty(nnz, np.int32); w = np.empty(nnz)
    _check(ctx, ctx.lib.topt_b200_filter_csr(h, _ptr(rp), _ptr(col), _ptr(w)))
    return FilterKernel(n, radius, rp, col, w, grid, h, ctx)


def _filter_product(kernel: FilterKernel, v, transpose: bool, what: str):
    n = kernel.size
    dev = _is_torch_cuda(v)
    size = v.numel() if dev else np.asarray(v).size
    if size != n:
        raise DomainError(f"{what}: field size does not match kernel")
    ctx = kernel._ctx or L.context(0)
    if dev:
        if kernel._h is None:
            raise DomainError(f"{what}: device fields need a kernel from build_filter")
        v = _dev_f64(v, what, n)
        import torch
        out = torch.empty_like(v)
        with ctx.ordered_with_torch():
            _check(ctx, ctx.lib.topt_b200_filter_apply_dev(ctx.h, kernel._h, int(transpose),
                                                           v.data_ptr(), out.data_ptr()))
        return out
    v = np.ascontiguousarray(v, np.float64)
    out = np.empty(n)
    if kernel._h is not None:
        _check(ctx, ctx.lib.topt_b200_filter_apply(ctx.h, kernel._h, int(transpose), _ptr(v),
                                                   _ptr(out)))
    else:
        rp = np.ascontiguousarray(kernel.row_ptr, np.int32)
        col = np.ascontiguousarray(kernel.col, np.int32)
        w = np.ascontiguousarray(kernel.weight, np.float64)
        _check(ctx, ctx.lib.topt_b200_csr_apply(ctx.h, n, _ptr(rp), _ptr(col), _ptr(w),
                                                int(transpose), _ptr(v), _ptr(out)))
    return out


def apply_filter(kernel: FilterKernel, raw):
    """filtered = W raw (filter.cpp:45-56)."""
    return _filter_product(kernel, raw, False, "apply_filter")


def filter_chain_rule(kernel: FilterKernel, grad_wrt_filtered):
    """W^T grad (filter.cpp:58-69)."""
    return _filter_product(kernel, grad_wrt_filtered, True, "filter_chain_rule")


@dataclasses.dataclass
class MaterialModel:
    """material.hpp:13-24 (SIMP)."""
    young_moduli: Sequence[float] = (1.0,)
    e_min: float = 1e-9
    poisson: float = 0.3
    penalty: float = 3.0

    def num_materials(self) -> int:
        return len(self.young_moduli)

    def validate(self):   # material.cpp:9-17
        if not len(self.young_moduli):
            raise ParameterError("material: no young moduli")
        if not (self.e_min > 0.0):
            raise ParameterError("material: e_min must be > 0")
        for e in self.young_moduli:
            if not (e > self.e_min):
                raise ParameterError("material: every E_j must exceed e_min")
        if not (0.0 < self.poisson < 0.5):
            raise ParameterError("material: poisson must lie in (0, 0.5)")
        if not (self.penalty >= 1.0):
            raise ParameterError("material: penalty must be >= 1")


@dataclasses.dataclass
class StiffnessInterpolation:
    moduli: object       # N
    derivative: object   # N*K channel-major


def interpolate_stiffness(densities, num_elements: int, model: MaterialModel,
                          device: int = 0) -> StiffnessInterpolation:
    """interpolate_stiffness (material.cpp:19-46) on the GPU.  Host arrays are
    copied in and out; torch CUDA tensors stay on the device."""
    import torch
    model.validate()
    k = model.num_materials()
    dev = _is_torch_cuda(densities)
    d = (_dev_f64(densities, "densities") if dev
         else torch.from_numpy(np.ascontiguousarray(densities, np.float64)).cuda(device))
    if d.numel() != num_elements * k:
        raise DomainError("interpolate_stiffness: density vector size mismatch")
    ctx = L.context(device)
    mod = torch.empty(num_elements, dtype=torch.float64, device=d.device)
    der = torch.empty(num_elements * k, dtype=torch.float64, device=d.device)
    young = np.ascontiguousarray(model.young_moduli, np.float64)
    with ctx.ordered_with_torch():
        rc = ctx.lib.topt_b200_interpolate_stiffness_dev(
            ctx.h, num_elements, k, _ptr(young), model.e_min, model.poisson, model.penalty,
            d.data_ptr(), mod.data_ptr(), der.data_ptr())
    if rc == L.ERR_DOMAIN:
        raise DomainError("interpolate_stiffness: density outside [0,1]")
    _check(ctx, rc)
    torch.cuda.synchronize(d.device)
    if dev:
        return StiffnessInterpolation(mod, der)
    return StiffnessInterpolation(mod.cpu().numpy(), der.cpu().numpy())


def element_stiffness_q4(poisson: float, element_size: float) -> np.ndarray:
    """element_stiffness_q4 (fea.cpp:20-58): the unit-modulus plane-stress Q4
    element matrix (8 x 8)."""
    lib = L.load()
    ke = np.empty(64)
    if lib.topt_b200_element_stiffness_q4(float(poisson), float(element_size), _ptr(ke)):
        raise ParameterError("element_stiffness_q4: poisson must lie in (0, 0.5) and "
                             "element_size > 0")
    return ke.reshape(8, 8)


def compliance_gradient(grid: StructuredGrid, displacement, derivative, model: MaterialModel,
                        device: int = 0):
    """Element energies u_e^T k0 u_e and the compliance gradient -dE * energy
    (fea.cpp:162-181) from a displacement field (all 2 (nx+1)(ny+1) dofs) and
    interpolate_stiffness's derivative.  Returns (energy, gradient)."""
    import torch
    k = model.num_materials()
    n = grid.num_elements()
    dev = _is_torch_cuda(displacement)
    cu = (lambda a, nm, sz: _dev_f64(a, nm, sz)) if dev else \
        (lambda a, nm, sz: torch.from_numpy(np.ascontiguousarray(a, np.float64)).cuda(device))
    u = cu(displacement, "displacement", grid.num_dofs())
    der = cu(derivative, "derivative", n * k)
    if u.numel() != grid.num_dofs() or der.numel() != n * k:
        raise DomainError("compliance_gradient: size mismatch")
    ctx = L.context(device)
    energy = torch.empty(n, dtype=torch.float64, device=u.device)
    grad = torch.empty(n * k, dtype=torch.float64, device=u.device)
    with ctx.ordered_with_torch():
        _check(ctx, ctx.lib.topt_b200_compliance_gradient_dev(
            ctx.h, grid.nx, grid.ny, grid.element_size, model.poisson, u.data_ptr(), k,
            der.data_ptr(), energy.data_ptr(), grad.data_ptr()))
    torch.cuda.synchronize(u.device)
    if dev:
        return energy, grad
    return energy.cpu().numpy(), grad.cpu().numpy()


def pgd_step_lockstep(slabs, n_global: int, settings: PgdSettings = None, device: int = 0,
                      row_counts=None):
    """One PGD step over element slabs, one lockstep rank per slab in this
    process (topt_b200_pgd_step_lockstep): the multi-rank data plane -- rank
    slabs, per-rank pass kernels, rank-order combine of the exchanged totals,
    replicated control -- with device copies instead of NCCL.  `slabs`: per
    rank a dict of torch CUDA tensors x, x_prev, g, g_prev, d_prev, grad (m x
    slab) and the shared g_values, bounds_g, is_equality, t, violation.
    Returns per-rank StepResults."""
    import torch
    world = len(slabs)
    settings = settings or PgdSettings()
    ctxs = [L.Context(device, r, world, lockstep=True) for r in range(world)]
    probs = (L.StepProblem * world)()
    outs = (L.StepOutputs * world)()
    metas = (L.ProjMeta * world)()
    keep, res_bufs = [], []
    for r, s in enumerate(slabs):
        n = int(s["x"].numel())
        m = int(len(s["g_values"]))
        pr = probs[r]
        pr.n, pr.m, pr.t, pr.violation = n, m, int(s.get("t", 1)), float(s.get("violation", 0.0))
        pr.lower, pr.upper = float(s.get("lower", 0.0)), float(s.get("upper", 1.0))
        arrs = {k: _dev_f64(s[k], k, n) for k in ("x", "x_prev", "g", "g_prev", "d_prev")}
        arrs["grad"] = _dev_f64(s["grad"], "grad", m * n)
        for k, a in arrs.items():
            setattr(pr, k, a.data_ptr())
        gv = np.ascontiguousarray(s["g_values"], np.float64)
        bg = np.ascontiguousarray(s["bounds_g"], np.float64)
        ie = (None if s.get("is_equality") is None
              else np.ascontiguousarray(s["is_equality"], np.uint8))
        pr.g_values, pr.bounds_g, pr.is_equality = _ptr(gv), _ptr(bg), _ptr(ie)
        pr.part_offsets = pr.part_indices = pr.owner = None
        b = {k: torch.empty(n, dtype=torch.float64, device=arrs["x"].device)
             for k in ("x_new", "d", "rho_tilde")}
        b.update(y=np.zeros(m), sl=np.zeros(m), gh=np.zeros(m))
        o = outs[r]
        o.x_new, o.d, o.rho_tilde = b["x_new"].data_ptr(), b["d"].data_ptr(), b["rho_tilde"].data_ptr()
        o.delta = o.mask = None
        o.y, o.slacks, o.g_hat = _ptr(b["y"]), _ptr(b["sl"]), _ptr(b["gh"])
        keep += [arrs, gv, bg, ie]
        res_bufs.append(b)
    handles = (C.c_void_p * world)(*[c.h for c in ctxs])
    rc_arr = None if row_counts is None else np.ascontiguousarray(row_counts, np.int64)
    opts = settings.options()._c()
    sc = settings._c()
    torch.cuda.current_stream(device).synchronize()   # the slabs' producers (own streams below)
    rc = ctxs[0].lib.topt_b200_pgd_step_lockstep(world, handles, probs, int(n_global), _ptr(rc_arr),
                                                 C.byref(sc), C.byref(opts), outs, metas)
    if rc != L.OK:
        msg = "; ".join(c.last_error() for c in ctxs if c.last_error())
        raise _ERRMAP.get(rc, RuntimeError)(msg)
    out = []
    for r in range(world):
        b, meta = res_bufs[r], metas[r]
        m = len(b["y"])
        proj = _meta_to_result(meta, None, b["y"].copy(), b["sl"].copy(), m)
        out.append(StepResult(x_new=b["x_new"], d=b["d"], rho_tilde=b["rho_tilde"], delta=None,
                              y=b["y"].copy(), slacks=b["sl"].copy(), g_hat=b["gh"].copy(),
                              alpha=meta.alpha, beta=meta.beta, fallback=bool(meta.fallback),
                              projection=proj))
    for c in ctxs:
        c.close()
    return out


# ---- FE solve and compliance sensitivities (fea.hpp:14-54, grid.hpp:36-45) -----
@dataclasses.dataclass
class BoundaryConditions:
    """grid.hpp:36-41: fixed dofs (sorted, unique) and point loads {dof: force}."""
    fixed_dofs: Sequence[int] = ()
    loads: dict = dataclasses.field(default_factory=dict)


def cantilever_bc(grid: StructuredGrid, load_magnitude: float = 1.0) -> BoundaryConditions:
    """grid.cpp:40-51: left edge clamped, downward unit load at the midpoint of
    the right edge (iy = ny / 2, rounded down)."""
    fixed = []
    for iy in range(grid.ny + 1):
        nd = iy * (grid.nx + 1)
        fixed += [2 * nd, 2 * nd + 1]
    tip = (grid.ny // 2) * (grid.nx + 1) + grid.nx
    return BoundaryConditions(sorted(fixed), {2 * tip + 1: -load_magnitude})


@dataclasses.dataclass
class SolveOptions:
    """fea.hpp:20-25.  The GPU solve is always the matrix-free PCG (the
    reference switches to a dense LDLT below dense_threshold free dofs; both
    meet the same relative-residual contract)."""
    rel_tolerance: float = 1e-8
    dense_threshold: int = 200
    force_iterative: bool = False


@dataclasses.dataclass
class LinearSystem:
    """fea.hpp:27-34 without the assembled matrix (the GPU never forms it)."""
    solution: object
    free_dofs: np.ndarray
    iterations: int
    residual: float


def assemble_and_solve(grid: StructuredGrid, bc: BoundaryConditions, element_moduli,
                       poisson: float = 0.3, options: SolveOptions = None,
                       device: int = 0) -> LinearSystem:
    """assemble_and_solve (fea.cpp:60-144) on the GPU: matrix-free Jacobi-PCG."""
    import torch
    options = options or SolveOptions()
    n = grid.num_elements()
    dev = _is_torch_cuda(element_moduli)
    E = (_dev_f64(element_moduli, "element_moduli") if dev
         else torch.from_numpy(np.ascontiguousarray(element_moduli, np.float64)).cuda(device))
    if E.numel() != n:
        raise DomainError("assemble_and_solve: element_moduli size mismatch")
    ctx = L.context(device)
    fixed = np.ascontiguousarray(sorted(bc.fixed_dofs), np.int32)
    ld = np.ascontiguousarray(list(bc.loads.keys()), np.int32)
    lv = np.ascontiguousarray(list(bc.loads.values()), np.float64)
    u = torch.empty(grid.num_dofs(), dtype=torch.float64, device=E.device)
    its = C.c_int64(0)
    res = C.c_double(0.0)
    with ctx.ordered_with_torch():
        rc = ctx.lib.topt_b200_fe_solve_dev(ctx.h, grid.nx, grid.ny, grid.element_size, poisson,
                                            E.data_ptr(), _ptr(fixed), len(fixed), _ptr(ld),
                                            _ptr(lv), len(ld), options.rel_tolerance,
                                            u.data_ptr(), C.byref(its), C.byref(res))
    if rc == L.ERR_PARAMETER:
        raise ParameterError("bc: invalid boundary conditions (no fixed dofs, out of range, "
                             "or a load on a fixed dof)")
    if rc == L.ERR_SINGULAR:
        raise SingularSystemError(f"assemble_and_solve: cg stalled at relative residual "
                                  f"{res.value:g} (system may be near-singular; check e_min)")
    _check(ctx, rc)
    mask = np.ones(grid.num_dofs(), bool)
    mask[fixed] = False
    sol = u if dev else u.cpu().numpy()
    return LinearSystem(sol, np.nonzero(mask)[0].astype(np.int32), int(its.value), float(res.value))


@dataclasses.dataclass
class ComplianceResult:
    compliance: float
    gradient: object
    solver_iterations: int


def compliance_and_gradient(grid: StructuredGrid, bc: BoundaryConditions, densities,
                            model: MaterialModel, options: SolveOptions = None,
                            device: int = 0) -> ComplianceResult:
    """compliance_and_gradient (fea.cpp:146-182), every stage on the GPU:
    SIMP interpolation, the FE solve, f.u and -dE * u_e^T k0 u_e."""
    import torch
    dev = _is_torch_cuda(densities)
    d = densities if dev else torch.from_numpy(np.ascontiguousarray(densities, np.float64)).cuda(device)
    interp = interpolate_stiffness(d, grid.num_elements(), model, device)
    sys_ = assemble_and_solve(grid, bc, interp.moduli, model.poisson, options, device)
    u = sys_.solution
    uh = u.cpu().numpy()
    comp = 0.0
    for dof, val in bc.loads.items():   # fea.cpp:157
        comp += val * uh[dof]
    _, grad = compliance_gradient(grid, u, interp.derivative, model, device)
    return ComplianceResult(comp, grad if dev else grad.cpu().numpy() if hasattr(grad, "cpu") else grad,
                            sys_.iterations)
