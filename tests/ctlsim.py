"""Python driver of tests/cpp/libctlsim.so (TEST HARNESS): runs the product
controller on the host with CPU-evaluated pass totals, optionally split over
R rank slabs (partials summed in rank order, as the multi-GPU path does)."""
import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "cpp", "libctlsim.so")
JOB_PROJECT, JOB_PGD_STEP = 0, 1
PH_DONE = 6
PATHS = {0: "single_binary", 1: "independent_binary", 2: "newton"}

_lib = None


def lib():
    global _lib
    if _lib is None:
        subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cpp")], check=True)
        _lib = C.CDLL(SO)
        _lib.sim_plan_size.restype = C.c_int64
        vp, d, i32, i64 = C.c_void_p, C.c_double, C.c_int, C.c_int64
        _lib.sim_setup.argtypes = [vp, i32, i32, i64, i64, i32] + [vp] * 16 + [d, d, i32, d, d]
        _lib.sim_partials.argtypes = [vp, vp]
        _lib.sim_consume.argtypes = [vp, vp]
        _lib.sim_phase.argtypes = [vp]
        _lib.sim_nslots.argtypes = [vp]
        _lib.sim_slot_op.argtypes = [vp, i32]
        _lib.sim_result.argtypes = [vp, vp, vp, vp, vp]
        _lib.sim_walk.argtypes = [vp, i32, vp, vp, vp]
        _lib.sim_set_hint.argtypes = [vp, i32, d, d]
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


class Rank:
    """One rank's slab [lo, hi) of a synth.StepProblem (host buffers)."""

    def __init__(self, prob, lo, hi, job=JOB_PGD_STEP, rho=None, gd=None, ghat=None):
        L = lib()
        self.plan = (C.c_char * L.sim_plan_size())()
        n = hi - lo
        m = prob.m
        self.keep = []
        sl = lambda a: np.ascontiguousarray(a[lo:hi], np.float64)  # noqa: E731
        self.x, self.xp, self.g, self.gp, self.dp = (sl(prob.x), sl(prob.x_prev), sl(prob.g),
                                                     sl(prob.g_prev), sl(prob.d_prev))
        self.grad = np.ascontiguousarray(prob.grad[:, lo:hi])
        self.rho = sl(rho) if rho is not None else np.zeros(n)
        self.gd = sl(gd) if gd is not None else None
        self.d = np.zeros(n); self.delta = np.zeros(n); self.xn = np.zeros(n)
        self.owner = None
        if prob.partition is not None and m > 1:
            own = np.full(prob.n, -1, np.int8)
            for j, p in enumerate(prob.partition):
                own[np.asarray(p)] = j
            self.owner = np.ascontiguousarray(own[lo:hi])
        self.Gmg = np.ascontiguousarray(prob.bounds_g - prob.g_values, np.float64)
        self.ghat = None if ghat is None else np.ascontiguousarray(ghat, np.float64)
        self.iseq = np.ascontiguousarray(prob.is_eq, np.int32)
        cnt = (np.array([len(p) for p in prob.partition], np.float64)
               if (prob.partition is not None and m > 1) else np.full(m, float(prob.n)))
        self.cnt = cnt
        L.sim_setup(self.plan, job, 0, n, prob.n, m, _p(self.x), _p(self.xp), _p(self.g),
                    _p(self.gp), _p(self.dp), _p(self.grad), _p(self.gd), _p(self.owner),
                    _p(self.rho), _p(self.d), _p(self.delta), _p(self.xn), _p(self.Gmg),
                    _p(self.ghat), _p(self.iseq), _p(cnt), prob.lower, prob.upper, prob.t,
                    prob.violation, float(n + 64))

    def phase(self):
        return lib().sim_phase(self.plan)

    def partials(self):
        ns = lib().sim_nslots(self.plan)
        out = np.zeros(max(ns, 1))
        lib().sim_partials(self.plan, _p(out))
        return out[:ns]

    def ops(self, ns):
        return [lib().sim_slot_op(self.plan, s) for s in range(ns)]

    def consume(self, totals):
        t = np.ascontiguousarray(totals, np.float64)
        if t.size == 0:
            t = np.zeros(1)
        lib().sim_consume(self.plan, _p(t))

    def walk(self, j):
        w = np.zeros(14); cand = np.zeros(64); nc = C.c_int(0)
        lib().sim_walk(self.plan, j, _p(w), _p(cand), C.byref(nc))
        return w, cand[:nc.value]

    def result(self, m):
        iv = np.zeros(10, np.int32); dv = np.zeros(4); y = np.zeros(m); gh = np.zeros(m)
        lib().sim_result(self.plan, _p(iv), _p(dv), _p(y), _p(gh))
        return dict(status=int(iv[0]), path=PATHS.get(int(iv[1])), newton_iters=int(iv[2]),
                    converged=bool(iv[3]), passes=int(iv[5]), sweeps=int(iv[6]),
                    stage1_row=int(iv[7]), near_ties=int(iv[8]), residual=dv[0],
                    alpha=dv[1], beta=dv[2], min_margin=dv[3], y=y, ghat=gh)


def combine(parts, ops):
    """Fixed rank-order combine of per-rank partial vectors."""
    tot = np.array(parts[0], copy=True)
    for p in parts[1:]:
        for s, o in enumerate(ops):
            tot[s] = tot[s] + p[s] if o == 0 else (min(tot[s], p[s]) if o == 1
                                                    else max(tot[s], p[s]))
    return tot


def bounds(n, R):
    return [(r * n // R, (r + 1) * n // R) for r in range(R)]


def run(prob, R=1, job=JOB_PGD_STEP, rho=None, gd=None, ghat=None, max_passes=4096,
        verbose=False, hints=None):
    ranks = [Rank(prob, lo, hi, job, rho, gd, ghat) for lo, hi in bounds(prob.n, R)]
    for j, h in enumerate(hints or []):
        if h is not None:
            for rk in ranks:
                lib().sim_set_hint(rk.plan, j, h[0], h[1])
    passes = 0
    while ranks[0].phase() != PH_DONE and passes < max_passes:
        if verbose:
            for j in range(prob.m):
                w, cand = ranks[0].walk(j)
                print(f"  pass {passes} phase {ranks[0].phase()} row {j}: lo {w[0]:.6g} hi {w[1]:.6g} "
                      f"ym {w[2]:.6g} yL {w[3]:.6g} yH {w[4]:.6g} it {int(w[5])} st {int(w[6])} "
                      f"direct {int(w[8])} E {w[7]:.3g}")
                if len(cand):
                    rk = ranks[0]
                    a = rk.grad[j]; lo_ = prob.lower - rk.rho; hi_ = prob.upper - rk.rho
                    def cls(y):
                        v = y * a
                        return np.where(v < lo_, 0, np.where(v > hi_, 2, 1))
                    act = int(np.count_nonzero((cls(w[9]) != cls(w[10])) & (a != 0)))
                    print(f"     window [{w[9]:.9g}, {w[10]:.9g}] active {act}  est kind {int(w[11])} ye {w[12]:.9g} sig {w[13]:.3g}")
                    print("     cand", " ".join(f"{c:.9g}" for c in cand))
        parts = [rk.partials() for rk in ranks]
        ops = ranks[0].ops(len(parts[0]))
        tot = combine(parts, ops)
        for rk in ranks:
            rk.consume(tot)
        passes += 1
    res = ranks[0].result(prob.m)
    res["x_new"] = np.concatenate([rk.xn for rk in ranks])
    res["d"] = np.concatenate([rk.d for rk in ranks])
    res["rho"] = np.concatenate([rk.rho for rk in ranks])
    for rk in ranks[1:]:
        assert np.array_equal(rk.result(prob.m)["y"], res["y"])  # replicated decisions
    return res
