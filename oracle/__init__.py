"""CPU checkers for the PGD-TO step — TEST INFRASTRUCTURE ONLY.

Two libraries, both loaded through ctypes:

* ``liboracle.so``  — oracle.c, a plain-C restatement of
  /root/reference/proj/src/projection.cpp and of SPEC.md's optimizer step.
* ``_ref/libtopt_ref.so`` — the reference's own projection.cpp compiled in
  place (oracle/Makefile) against the Eigen-subset shim; present wherever it
  was built (it travels to the GPU box as a prebuilt file).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` arm may import this package; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtopt_ref.so")

PATHS = {0: "single_binary", 1: "independent_binary", 2: "newton"}
ERRS = {0: None, 1: "ParameterError", 2: "DomainError", 3: "SingularSystemError",
        4: "InfeasibleLinearization", 5: "NumericalError", 6: "UnsupportedProblem",
        99: "std::exception"}

_dp = C.POINTER(C.c_double)
_i64 = C.c_int64


class OrcOpts(C.Structure):
    _fields_ = [("c", C.c_double), ("tol_b", C.c_double), ("tol_n", C.c_double),
                ("newton_maxiter", C.c_int), ("binary_maxiter", C.c_int)]


class OrcMeta(C.Structure):
    _fields_ = [("path", C.c_int), ("newton_iters", C.c_int), ("converged", C.c_int),
                ("curvature_violations", C.c_int), ("stage1_row", C.c_int),
                ("residual", C.c_double), ("bisect_iters", C.c_int * 64),
                ("iter_trace", _dp)]


class OrcPgdSettings(C.Structure):
    _fields_ = [("alpha_max", C.c_double), ("alpha_fallback", C.c_double),
                ("omega", C.c_double), ("eps_alpha", C.c_double), ("tol_n", C.c_double),
                ("t_warmup", C.c_int)]


class OrcStepInfo(C.Structure):
    _fields_ = [("alpha", C.c_double), ("beta", C.c_double), ("fallback", C.c_int)]


def build(quiet: bool = True) -> None:
    """Compile liboracle.so (and oracle/_ref when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build()
        _lib = C.CDLL(ORACLE_SO)
        _lib.orc_spectral_step_size.restype = C.c_double
        _lib.orc_spectral_from_sums.restype = C.c_double
        _lib.orc_pr_beta.restype = C.c_double
        _lib.orc_pr_beta_from_sums.restype = C.c_double
        _lib.orc_trace_len.restype = C.c_int64
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference)")
        _ref = C.CDLL(REF_SO)
    return _ref


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _opts(c=1e12, tol_b=1e-8, tol_n=1e-6, newton_maxiter=50, binary_maxiter=200):
    return OrcOpts(c, tol_b, tol_n, newton_maxiter, binary_maxiter)


def _part(partition, m):
    if partition is None:
        return None, None
    off = np.zeros(m + 1, np.int64)
    for j, p in enumerate(partition):
        off[j + 1] = off[j] + len(p)
    idx = (np.concatenate([np.asarray(p, np.int32) for p in partition])
           if len(partition) else np.zeros(0, np.int32))
    return off, np.ascontiguousarray(idx, np.int32)


class OracleError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"{ERRS.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERRS.get(code, str(code))


# ----------------------------------------------------------------------------
# The restatement (oracle.c)
# ----------------------------------------------------------------------------

def build_ghat(grad, g_values, bounds_g, gd_step):
    grad = _f64(grad); m, n = grad.shape
    out = np.empty(m)
    lib().orc_build_ghat(_i64(n), _i64(m), _p(grad), _p(_f64(g_values)), _p(_f64(bounds_g)),
                         _p(_f64(gd_step)), _p(out))
    return out


def delta_of_y(y, grad, rho, lower=0.0, upper=1.0):
    grad = _f64(grad); m, n = grad.shape
    out = np.empty(n)
    lib().orc_delta_of_y(_i64(n), _i64(m), _p(_f64(y)), _p(grad), _p(_f64(rho)),
                         C.c_double(lower), C.c_double(upper), _p(out))
    return out


def residual_h(y, grad, ghat, rho, lower=0.0, upper=1.0, c=1e12):
    grad = _f64(grad); m, n = grad.shape
    out = np.empty(m)
    rc = lib().orc_residual_h(_i64(n), _i64(m), _p(_f64(y)), _p(grad), _p(_f64(ghat)),
                              _p(_f64(rho)), C.c_double(lower), C.c_double(upper),
                              C.c_double(c), _p(out))
    if rc:
        raise OracleError(rc)
    return out


def project(rho, grad, g_values, bounds_g, gd_step, is_eq=None, partition=None,
            lower=0.0, upper=1.0, which="auto", trace=False, **opts):
    """oracle.c project / project_* ; returns a dict like ProjectionResult."""
    grad = _f64(grad); m, n = grad.shape
    rho = _f64(rho)
    is_eq = np.zeros(m, np.uint8) if is_eq is None else np.ascontiguousarray(is_eq, np.uint8)
    ghat = build_ghat(grad, g_values, bounds_g, gd_step)
    off, idx = _part(partition, m)
    delta = np.empty(n); y = np.empty(m); sl = np.empty(m)
    meta = OrcMeta()
    gam = np.zeros(128)
    meta.iter_trace = gam.ctypes.data_as(_dp)
    o = _opts(**opts)
    tbuf = None
    if trace:
        tbuf = np.zeros(4 * 200000)
        lib().orc_trace_set(_p(tbuf), _i64(tbuf.size))
    L = lib()
    common = (C.c_double(lower), C.c_double(upper))
    if which == "auto":
        rc = L.orc_project(_i64(n), _i64(m), _p(rho), _p(grad), _p(_f64(g_values)),
                           _p(_f64(bounds_g)), _p(_f64(gd_step)), _p(ghat), _p(is_eq), _p(off),
                           _p(idx), *common, C.byref(o), _p(delta), _p(y), _p(sl),
                           C.byref(meta))
    elif which == "single":
        rc = L.orc_project_single(_i64(n), _i64(m), _p(rho), _p(grad), _p(ghat), _p(is_eq),
                                  *common, C.c_double(o.tol_b), C.c_int(o.binary_maxiter),
                                  _p(delta), _p(y), _p(sl), C.byref(meta))
    elif which == "independent":
        rc = L.orc_project_independent(_i64(n), _i64(m), _p(rho), _p(grad), _p(_f64(g_values)),
                                       _p(_f64(bounds_g)), _p(_f64(gd_step)), _p(ghat),
                                       _p(is_eq), _p(off), _p(idx), *common,
                                       C.c_double(o.tol_b), C.c_int(o.binary_maxiter),
                                       _p(delta), _p(y), _p(sl), C.byref(meta))
    elif which == "newton":
        rc = L.orc_project_newton(_i64(n), _i64(m), _p(rho), _p(grad), _p(ghat), _p(is_eq),
                                  *common, C.byref(o), _p(delta), _p(y), _p(sl),
                                  C.byref(meta))
    else:
        raise ValueError(which)
    tr = None
    if trace:
        k = int(L.orc_trace_len())
        tr = tbuf[:k].reshape(-1, 4).copy()
        L.orc_trace_set(None, _i64(0))
    if rc:
        raise OracleError(rc)
    return dict(delta=delta, y=y, slacks=sl, path=PATHS[meta.path],
                newton_iters=meta.newton_iters, residual=meta.residual,
                converged=bool(meta.converged), curvature_violations=meta.curvature_violations,
                stage1_row=meta.stage1_row, ghat=ghat,
                bisect_iters=list(meta.bisect_iters[:m]) if m <= 64 else None,
                gammas=gam[:min(meta.newton_iters, 64)].copy(),
                phi_inf=gam[64:64 + min(meta.newton_iters, 64)].copy(), trace=tr)


def enum_project(rho, grad, ghat, is_eq=None, lower=0.0, upper=1.0, tol=1e-10):
    """SPEC.md:231-239 enumeration oracle (oracle/enum.c): exact projection by
    enumerating 3^N box x 2^m constraint activity patterns.  Returns (delta, y)
    or None when the linearized set is empty."""
    grad = _f64(np.atleast_2d(grad)); m, n = grad.shape
    is_eq = np.zeros(m, np.uint8) if is_eq is None else np.ascontiguousarray(is_eq, np.uint8)
    d = np.empty(n); y = np.empty(m)
    rc = lib().orc_enum_project(C.c_int(n), C.c_int(m), _p(_f64(rho)), _p(grad), _p(_f64(ghat)),
                                _p(is_eq), C.c_double(lower), C.c_double(upper), C.c_double(tol),
                                _p(d), _p(y))
    if rc == 2:
        raise ValueError("enumeration oracle: N <= 12 and m <= 3 only")
    return None if rc == 1 else (d, y)


# ---- upstream of the step ------------------------

def filter_csr(nx, ny, radius):
    """oracle/upstream.c restatement of build_filter (filter.cpp:10-43)."""
    L = lib()
    L.orc_filter_csr.restype = C.c_int64
    nnz = L.orc_filter_csr(C.c_int(nx), C.c_int(ny), C.c_double(radius), None, None, None)
    rp = np.empty(nx * ny + 1, np.int32); col = np.empty(nnz, np.int32); w = np.empty(nnz)
    L.orc_filter_csr(C.c_int(nx), C.c_int(ny), C.c_double(radius), _p(rp), _p(col), _p(w))
    return rp, col, w


def filter_apply(nx, ny, radius, x, transpose=False):
    out = np.empty(nx * ny)
    lib().orc_filter_apply(C.c_int(nx), C.c_int(ny), C.c_double(radius), C.c_int(int(transpose)),
                           _p(_f64(x)), _p(out))
    return out


def interpolate(dens, n, young, e_min=1e-9, penalty=3.0):
    k = len(young)
    mod = np.empty(n); der = np.empty(n * k)
    rc = lib().orc_interpolate(_i64(n), C.c_int(k), _p(_f64(young)), C.c_double(e_min),
                               C.c_double(penalty), _p(_f64(dens)), _p(mod), _p(der))
    if rc:
        raise OracleError(2, "interpolate_stiffness: density outside [0,1]")
    return mod, der


def element_q4(poisson=0.3, h=1.0):
    ke = np.empty(64)
    lib().orc_element_q4(C.c_double(poisson), C.c_double(h), _p(ke))
    return ke.reshape(8, 8)


def energy_gradient(nx, ny, u, der, k=1, poisson=0.3, h=1.0):
    n = nx * ny
    e = np.empty(n); g = np.empty(n * k)
    lib().orc_energy_gradient(C.c_int(nx), C.c_int(ny), C.c_double(h), C.c_double(poisson),
                              _p(_f64(u)), C.c_int(k), _p(_f64(der)), _p(e), _p(g))
    return e, g


def ref_filter_csr(nx, ny, radius):
    """The reference's own build_filter (oracle/_ref)."""
    nnz = np.array([0], np.int64)
    err = C.create_string_buffer(512)
    rc = ref().ref_filter_csr(C.c_int(nx), C.c_int(ny), C.c_double(radius), None, None, None,
                              _p(nnz), err, C.c_size_t(512))
    if rc:
        raise OracleError(rc, err.value.decode())
    rp = np.empty(nx * ny + 1, np.int32); col = np.empty(int(nnz[0]), np.int32)
    w = np.empty(int(nnz[0]))
    ref().ref_filter_csr(C.c_int(nx), C.c_int(ny), C.c_double(radius), _p(rp), _p(col), _p(w),
                         _p(nnz), err, C.c_size_t(512))
    return rp, col, w


def ref_filter_apply(nx, ny, radius, x, transpose=False):
    out = np.empty(nx * ny)
    err = C.create_string_buffer(512)
    rc = ref().ref_filter_apply(C.c_int(nx), C.c_int(ny), C.c_double(radius),
                                C.c_int(int(transpose)), _p(_f64(x)), _p(out), err,
                                C.c_size_t(512))
    if rc:
        raise OracleError(rc, err.value.decode())
    return out


def ref_interpolate(dens, n, young, e_min=1e-9, poisson=0.3, penalty=3.0):
    k = len(young)
    mod = np.empty(n); der = np.empty(n * k)
    err = C.create_string_buffer(512)
    rc = ref().ref_interpolate(C.c_size_t(n), C.c_size_t(k), _p(_f64(young)), C.c_double(e_min),
                               C.c_double(poisson), C.c_double(penalty), _p(_f64(dens)),
                               _p(mod), _p(der), err, C.c_size_t(512))
    if rc:
        raise OracleError(rc, err.value.decode())
    return mod, der


def fe_system(nx, ny, moduli, fixed, loads, poisson=0.3, h=1.0):
    """assemble_and_solve's free-dof system (fea.cpp:60-104) restated with
    scipy.sparse: triplets E_e k0[i][j] over free dofs, summed duplicates;
    the right-hand side from the point loads.  Returns (K_free, f_free,
    free_dof_index)."""
    import scipy.sparse as sp
    nd = 2 * (nx + 1) * (ny + 1)
    fixed_mask = np.zeros(nd, bool)
    fixed_mask[np.asarray(fixed, np.int64)] = True
    dof_map = -np.ones(nd, np.int64)
    free = np.nonzero(~fixed_mask)[0]
    dof_map[free] = np.arange(free.size)
    ke = element_q4(poisson, h)
    rows, cols, vals = [], [], []
    for e in range(nx * ny):
        ex, ey = e % nx, e // nx
        n1 = ey * (nx + 1) + ex; n2 = n1 + 1; n3 = (ey + 1) * (nx + 1) + ex + 1; n4 = n3 - 1
        dofs = [2 * n1, 2 * n1 + 1, 2 * n2, 2 * n2 + 1, 2 * n3, 2 * n3 + 1, 2 * n4, 2 * n4 + 1]
        gi = dof_map[dofs]
        for i in range(8):
            if gi[i] < 0:
                continue
            for j in range(8):
                if gi[j] < 0:
                    continue
                rows.append(gi[i]); cols.append(gi[j]); vals.append(moduli[e] * ke[i, j])
    K = sp.csr_matrix((vals, (rows, cols)), shape=(free.size, free.size))
    f = np.zeros(free.size)
    for dof, val in loads.items():
        if dof_map[dof] >= 0:
            f[dof_map[dof]] += val
    return K, f, free


def fe_solve(nx, ny, moduli, fixed, loads, poisson=0.3, h=1.0):
    """Direct sparse solve of the reference's free-dof system (the oracle for
    the GPU's iterative solve): u on all dofs, fixed ones 0."""
    import scipy.sparse.linalg as sla
    K, f, free = fe_system(nx, ny, moduli, fixed, loads, poisson, h)
    u = np.zeros(2 * (nx + 1) * (ny + 1))
    u[free] = sla.spsolve(K.tocsc(), f)
    return u


def random_instance(rng, n, m, feasible=True, eq_rows=0):
    """A random projection instance (rho_tilde, A, g_hat): rho in (-0.3, 1.3),
    rows ~ N(0, 1); feasible ones get g_hat = A (x0 - rho) + slack for a random
    box point x0 (slack >= 0 on inequality rows, 0 on equality rows)."""
    rho = rng.uniform(-0.3, 1.3, n)
    A = rng.standard_normal((m, n))
    x0 = rng.uniform(0.0, 1.0, n)
    base = A @ (x0 - rho)
    slack = rng.uniform(0.0, 0.5, m) * (rng.uniform(size=m) < 0.7)
    is_eq = np.zeros(m, np.uint8)
    is_eq[:eq_rows] = 1
    slack[:eq_rows] = 0.0
    ghat = base + slack if feasible else base - 5.0 - abs(base)
    return rho, A, ghat, is_eq


def settings(alpha_max=1e2, alpha_fallback=0.2, omega=1.0, eps_alpha=1e-6, tol_n=1e-6,
             t_warmup=50):
    return OrcPgdSettings(alpha_max, alpha_fallback, omega, eps_alpha, tol_n, t_warmup)


def step_direction(x, x_prev, g, g_prev, d_prev, t=1, violation=0.0, **s):
    """Spec step (BB / PR+ / fallback / rho_tilde). Returns (d, gd_step, rho_tilde, info)."""
    x = _f64(x); n = x.size
    d = np.empty(n); gd = np.empty(n); rt = np.empty(n)
    st = OrcStepInfo()
    ss = settings(**s)
    lib().orc_step_direction(_i64(n), _p(x), _p(_f64(x_prev)), _p(_f64(g)), _p(_f64(g_prev)),
                             _p(_f64(d_prev)), C.c_int(t), C.c_double(violation),
                             C.byref(ss), _p(d), _p(gd), _p(rt), C.byref(st))
    return d, gd, rt, dict(alpha=st.alpha, beta=st.beta, fallback=bool(st.fallback))


def spectral_step_size(x, x_prev, g, g_prev, alpha_max=1e2, eps_alpha=1e-6):
    x = _f64(x)
    return lib().orc_spectral_step_size(_i64(x.size), _p(x), _p(_f64(x_prev)), _p(_f64(g)),
                                        _p(_f64(g_prev)), C.c_double(alpha_max),
                                        C.c_double(eps_alpha))


def pr_beta(g, g_prev):
    g = _f64(g)
    return lib().orc_pr_beta(_i64(g.size), _p(g), _p(_f64(g_prev)))


def pgd_step(prob, which="auto", trace=False, **opts):
    """Full oracle step on a synth.StepProblem: step direction + build + project."""
    d, gd, rt, info = step_direction(prob.x, prob.x_prev, prob.g, prob.g_prev, prob.d_prev,
                                     prob.t, prob.violation)
    res = project(rt, prob.grad, prob.g_values, prob.bounds_g, gd, prob.is_eq, prob.partition,
                  prob.lower, prob.upper, which=which, trace=trace, **opts)
    res.update(d=d, gd_step=gd, rho_tilde=rt, x_new=rt + res["delta"], **info)
    return res


# ----------------------------------------------------------------------------
# The compiled reference (oracle/_ref/libtopt_ref.so)
# ----------------------------------------------------------------------------

_WHICH = {"auto": 0, "single": 1, "independent": 2, "newton": 3}


def ref_project(rho, grad, g_values, bounds_g, gd_step, is_eq=None, partition=None,
                lower=0.0, upper=1.0, which="auto", c=1e12, tol_b=1e-8, tol_n=1e-6,
                newton_maxiter=50, binary_maxiter=200):
    grad = _f64(grad); m, n = grad.shape
    is_eq = None if is_eq is None else np.ascontiguousarray(is_eq, np.uint8)
    off, idx = _part(partition, m)
    delta = np.empty(n); y = np.empty(m); sl = np.empty(m); ghat = np.empty(m)
    meta = np.zeros(4, np.int32); resid = C.c_double(0.0)
    err = C.create_string_buffer(512)
    rc = ref().ref_project(C.c_int(_WHICH[which]), C.c_size_t(n), C.c_size_t(m),
                           _p(_f64(rho)), _p(grad), _p(_f64(g_values)), _p(_f64(bounds_g)),
                           _p(_f64(gd_step)), _p(is_eq), _p(off), _p(idx), C.c_double(lower),
                           C.c_double(upper), C.c_double(c), C.c_double(tol_b),
                           C.c_double(tol_n), C.c_int(newton_maxiter), C.c_int(binary_maxiter),
                           _p(delta), _p(y), _p(sl), _p(meta), C.byref(resid), _p(ghat), err,
                           C.c_size_t(512))
    if rc:
        raise OracleError(rc, err.value.decode())
    return dict(delta=delta, y=y, slacks=sl, path=PATHS[int(meta[0])],
                newton_iters=int(meta[1]), converged=bool(meta[2]),
                curvature_violations=int(meta[3]), residual=resid.value, ghat=ghat)


def ref_build_ghat(grad, g_values, bounds_g, gd_step, is_eq=None, partition=None):
    grad = _f64(grad); m, n = grad.shape
    off, idx = _part(partition, m)
    out = np.empty(m)
    err = C.create_string_buffer(512)
    rc = ref().ref_build_ghat(C.c_size_t(n), C.c_size_t(m), _p(grad), _p(_f64(g_values)),
                              _p(_f64(bounds_g)), _p(_f64(gd_step)),
                              _p(None if is_eq is None else np.ascontiguousarray(is_eq, np.uint8)),
                              _p(off), _p(idx), _p(out), err, C.c_size_t(512))
    if rc:
        raise OracleError(rc, err.value.decode())
    return out


def ref_delta_of_y(y, grad, rho, lower=0.0, upper=1.0):
    grad = _f64(grad); m, n = grad.shape
    out = np.empty(n)
    err = C.create_string_buffer(512)
    rc = ref().ref_delta_of_y(C.c_size_t(n), C.c_size_t(m), _p(_f64(y)), _p(grad),
                              _p(_f64(rho)), C.c_double(lower), C.c_double(upper), _p(out), err,
                              C.c_size_t(512))
    if rc:
        raise OracleError(rc, err.value.decode())
    return out


def ref_residual_h(y, grad, g_values, bounds_g, gd_step, rho, lower=0.0, upper=1.0, c=1e12):
    grad = _f64(grad); m, n = grad.shape
    out = np.empty(m)
    err = C.create_string_buffer(512)
    rc = ref().ref_residual_h(C.c_size_t(n), C.c_size_t(m), _p(_f64(y)), _p(grad),
                              _p(_f64(g_values)), _p(_f64(bounds_g)), _p(_f64(gd_step)),
                              _p(_f64(rho)), C.c_double(lower), C.c_double(upper),
                              C.c_double(c), _p(out), err, C.c_size_t(512))
    if rc:
        raise OracleError(rc, err.value.decode())
    return out


def ref_validate(grad, g_values, bounds_g, gd_step, ghat_override=None, partition=None):
    grad = _f64(grad); m, n = grad.shape
    off, idx = _part(partition, m)
    err = C.create_string_buffer(512)
    rc = ref().ref_validate(C.c_size_t(n), C.c_size_t(m), _p(grad), _p(_f64(g_values)),
                            _p(_f64(bounds_g)), _p(_f64(gd_step)),
                            _p(None if ghat_override is None else _f64(ghat_override)),
                            _p(off), _p(idx), err, C.c_size_t(512))
    if rc:
        raise OracleError(rc, err.value.decode())
