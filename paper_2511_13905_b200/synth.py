"""Seeded synthetic PGD-TO step inputs for BASELINE.json's five configs.

The FE solve and density filter are outside the hot path (BASELINE.json
`north_star`); these generators stand in for them with the distributions the
configs state.  Everything is numpy, seeded, and identical for any consumer
(GPU path, oracle, bench).  Choices the configs leave open are pinned here and
recorded in DESIGN.md §Workloads:

* t = 1 (spectral branch), x_prev = clip(x0 + N(0, 0.01^2), 0, 1), g_prev is
  recomputed from x_prev with the SAME e, d_prev = g_prev (d_0 = g_0).
* C2: objective gradient = unit volumes (g = g_prev = 1, so ||y|| = 0 and the
  BB step is alpha_max, beta = 0 -- the literal reading);
  C_lin = -c^T x0, g_value = C_lin, G = 1.1 C_lin.
* C3: 4 materials channel-major (material.hpp:28), row k = 1 on block k,
  partition = the 4 contiguous blocks, G_k = 0.1 N_el.
* Streams are chunked (CHUNK elements per Philox key) and the global sums use
  a fixed pairwise order, so any slab is generated alone and every host
  produces the same bits.
* C4/C5: element-unit centroids (idx + 0.5) h with h = 1 (grid.hpp:29-33),
  x fastest; rows [vol, +a_x, -a_x, +a_y, -a_y, +a_z, -a_z] with
  a = (c - R)/S, g = +-(R - L/2), G = 0.01.  `com_offset_x`
  shifts the x target (the C4'/C5' forced-Newton variant).
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np


@dataclasses.dataclass
class StepProblem:
    name: str
    n: int
    m: int
    x: np.ndarray
    x_prev: np.ndarray
    g: np.ndarray
    g_prev: np.ndarray
    d_prev: np.ndarray
    grad: np.ndarray          # (m, n) row-major constraint gradients A
    g_values: np.ndarray      # (m,)
    bounds_g: np.ndarray      # (m,)
    is_eq: np.ndarray         # (m,) uint8
    partition: Optional[list] = None   # list of int32 index arrays, or None
    lower: float = 0.0
    upper: float = 1.0
    t: int = 1
    violation: float = 0.0
    grid: tuple = ()
    rows: Optional[list] = None       # structured description of the rows (C4/C5)
    n_global: int = 0                 # elements of the whole design (0: = n)
    offset: int = 0                   # global index of element 0 of this slab

    def __post_init__(self):
        if not self.n_global:
            self.n_global = self.n

    @property
    def part_offsets(self):
        if self.partition is None:
            return None, None
        off = np.zeros(self.m + 1, dtype=np.int64)
        for j, p in enumerate(self.partition):
            off[j + 1] = off[j] + len(p)
        idx = (np.concatenate(self.partition).astype(np.int32)
               if self.m else np.zeros(0, np.int32))
        return off, idx


# Streams are drawn in CHUNK-element chunks, chunk c of stream s from its own
# Philox key (seed, s, c): any element range (a rank's slab) is generated
# without the rest, identically for every sharding.  Global reductions (the
# volume / COM / compliance constants) use a fixed blocked pairwise order of
# elementwise IEEE additions -- identical on every host (no BLAS, no SIMD-
# dependent reduction order).
CHUNK = 1 << 20


def _rng(seed: int, stream: int, chunk: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(np.random.SeedSequence([seed, stream, chunk])))


def _draw(seed, stream, n, fn, lo=0, hi=None):
    """Elements [lo, hi) of the length-n stream `stream` (fn(gen, k) draws k values)."""
    hi = n if hi is None else hi
    out = np.empty(max(hi - lo, 0))
    if hi <= lo:
        return out
    for c in range(lo // CHUNK, (hi - 1) // CHUNK + 1):
        b = c * CHUNK
        ln = min(CHUNK, n - b)
        v = fn(_rng(seed, stream, c), ln)
        s, e = max(lo, b), min(hi, b + ln)
        out[s - lo:e - lo] = v[s - b:e - b]
    return out


def _pw(v) -> float:
    """Pairwise sum by halving (zero-padded to a power of two): every step is an
    elementwise IEEE add, so the result is the same on every platform."""
    v = np.asarray(v, dtype=np.float64)
    if v.size == 0:
        return 0.0
    size = 1 << (int(v.size) - 1).bit_length()
    if size != v.size:
        v = np.concatenate([v, np.zeros(size - v.size)])
    while v.size > 1:
        v = v[0::2] + v[1::2]
    return float(v[0])


def det_sum(chunk_values) -> float:
    """Deterministic sum of a stream given chunk by chunk (CHUNK-aligned)."""
    return _pw([_pw(c) for c in chunk_values])


def _chunks(a):
    return (a[b:b + CHUNK] for b in range(0, a.size, CHUNK))


def _uniform(lo_v, hi_v):
    return lambda r, k: r.uniform(lo_v, hi_v, k)


def _normal(r, k):
    return r.standard_normal(k)


def _design(seed, n, lo, hi, stream0=0, slab=None):
    """x0 ~ U(lo, hi), e ~ LogNormal(0, 1), x_prev = clip(x0 + N(0, 0.01^2), 0, 1)
    on the slab [a, b) of the n-element design (default: all of it)."""
    a, b = slab if slab is not None else (0, n)
    x0 = _draw(seed, stream0, n, _uniform(lo, hi), a, b)
    e = np.exp(_draw(seed, stream0 + 1, n, _normal, a, b))        # LogNormal(0, 1)
    noise = _draw(seed, stream0 + 2, n, _normal, a, b) * 0.01
    x_prev = np.clip(x0 + noise, 0.0, 1.0)
    return x0, e, x_prev


def _x0_chunks(seed, n, lo, hi, stream0=0):
    """x0 of the WHOLE design, chunk by chunk (global sums on a slab rank)."""
    for c in range((n + CHUNK - 1) // CHUNK):
        b = c * CHUNK
        yield b, _rng(seed, stream0, c).uniform(lo, hi, min(CHUNK, n - b))


def min_compliance_volume(nx=256, ny=128, seed=1, volfrac=0.5, slab=None) -> StepProblem:
    """C1: single linear volume constraint, unit element volumes."""
    n = nx * ny
    a, b = slab if slab is not None else (0, n)
    x0, e, xp = _design(seed, n, 0.05, 0.95, slab=slab)
    g = -3.0 * x0 * x0 * e
    gp = -3.0 * xp * xp * e
    S = det_sum(c for _, c in _x0_chunks(seed, n, 0.05, 0.95))
    return StepProblem(
        name=f"C1_min_compliance_{nx}x{ny}", n=b - a, m=1, x=x0, x_prev=xp, g=g, g_prev=gp,
        d_prev=gp.copy(), grad=np.ones((1, b - a)), g_values=np.array([S]),
        bounds_g=np.array([volfrac * n]), is_eq=np.zeros(1, np.uint8), grid=(nx, ny),
        n_global=n, offset=a)


def min_volume_compliance(nx=1024, ny=1024, seed=2, factor=1.1, slab=None) -> StepProblem:
    """C2: min volume under a linearised compliance constraint (dense row)."""
    n = nx * ny
    a, b = slab if slab is not None else (0, n)
    x0, e, xp = _design(seed, n, 0.05, 0.95, slab=slab)
    c = -3.0 * x0 * x0 * e
    if slab is None:
        c_lin = -det_sum(_chunks(c * x0))
    else:   # the global linearised compliance needs every chunk's c . x0
        parts = []
        for bb, x0c in _x0_chunks(seed, n, 0.05, 0.95):
            ec = np.exp(_rng(seed, 1, bb // CHUNK).standard_normal(x0c.size))
            parts.append((-3.0 * x0c * x0c * ec) * x0c)
        c_lin = -det_sum(parts)
    ones = np.ones(b - a)
    return StepProblem(
        name=f"C2_min_volume_{nx}x{ny}", n=b - a, m=1, x=x0, x_prev=xp, g=ones,
        g_prev=ones.copy(), d_prev=ones.copy(), grad=c.reshape(1, b - a),
        g_values=np.array([c_lin]), bounds_g=np.array([factor * c_lin]),
        is_eq=np.zeros(1, np.uint8), grid=(nx, ny), n_global=n, offset=a)


def multi_material(nx=128, ny=128, nz=64, seed=3, n_mat=4, frac=0.1) -> StepProblem:
    """C3: n_mat materials, independent volume constraints (partitioned)."""
    ne = nx * ny * nz
    n = n_mat * ne
    xs, xps, gs, gps = [], [], [], []
    for k in range(n_mat):
        x0, e, xp = _design(seed, ne, 0.01, 0.24, stream0=10 * k)
        xs.append(x0); xps.append(xp)
        gs.append(-3.0 * x0 * x0 * e); gps.append(-3.0 * xp * xp * e)
    x0 = np.concatenate(xs); xp = np.concatenate(xps)
    g = np.concatenate(gs); gp = np.concatenate(gps)
    grad = np.zeros((n_mat, n))
    for k in range(n_mat):
        grad[k, k * ne:(k + 1) * ne] = 1.0
    part = [np.arange(k * ne, (k + 1) * ne, dtype=np.int32) for k in range(n_mat)]
    gv = np.array([det_sum(_chunks(xs[k])) for k in range(n_mat)])
    return StepProblem(
        name=f"C3_multi_material_{n_mat}x{nx}x{ny}x{nz}", n=n, m=n_mat, x=x0, x_prev=xp, g=g,
        g_prev=gp, d_prev=gp.copy(), grad=grad, g_values=gv,
        bounds_g=np.full(n_mat, frac * ne), is_eq=np.zeros(n_mat, np.uint8), partition=part,
        grid=(n_mat, nx, ny, nz))


def _centroids(nx, ny, b, k):
    """Element-unit centroids (idx + 0.5) of global elements [b, b + k), x fastest
    (grid.hpp:29-33 with h = 1)."""
    idx = np.arange(b, b + k, dtype=np.int64)
    return ((idx % nx) + 0.5, ((idx // nx) % ny) + 0.5, (idx // (nx * ny)) + 0.5)


def com_constrained(nx=256, ny=256, nz=128, seed=4, volfrac=0.3, band=0.01,
                    com_offset_x=0.0, slab=None) -> StepProblem:
    """C4/C5: volume + paired centre-of-mass rows (m = 7), coupled -> Newton."""
    n = nx * ny * nz
    a0, b0 = slab if slab is not None else (0, n)
    ln = b0 - a0
    x0, e, xp = _design(seed, n, 0.05, 0.95, slab=slab)
    g = -3.0 * x0 * x0 * e
    gp = -3.0 * xp * xp * e
    # global S = sum x0 and first moments sum c_a x0 (deterministic blocked order)
    ps, pm = [], ([], [], [])
    src = (_x0_chunks(seed, n, 0.05, 0.95) if slab is not None
           else ((bb, x0[bb:bb + CHUNK]) for bb in range(0, n, CHUNK)))
    for bb, x0c in src:
        ps.append(x0c)
        for ax, cc in enumerate(_centroids(nx, ny, bb, x0c.size)):
            pm[ax].append(_pw(cc * x0c))
    S = det_sum(ps)
    del ps
    Ms = [_pw(v) for v in pm]
    grad = np.empty((7, ln))
    gv = np.empty(7)
    G = np.empty(7)
    grad[0] = 1.0
    gv[0] = S
    G[0] = volfrac * n
    # the same rows, described (structured-row extension, api rows=...)
    rows = [dict(kind="const", value=1.0)]
    cs = _centroids(nx, ny, a0, ln)
    for ax, (c, L) in enumerate(zip(cs, (nx, ny, nz))):
        R = Ms[ax] / S
        target = L / 2.0 + (com_offset_x if ax == 0 else 0.0)
        row = (c - R) / S
        grad[1 + 2 * ax] = row
        grad[2 + 2 * ax] = -row
        gv[1 + 2 * ax] = R - target
        gv[2 + 2 * ax] = -(R - target)
        G[1 + 2 * ax] = band
        G[2 + 2 * ax] = band
        rows.append(dict(kind="centroid", axis=ax, center=R, scale=S, sign=1.0))
        rows.append(dict(kind="centroid", axis=ax, center=R, scale=S, sign=-1.0))
    del cs
    return StepProblem(
        name=f"C4_com_{nx}x{ny}x{nz}" + (f"_off{com_offset_x}" if com_offset_x else ""),
        n=ln, m=7, x=x0, x_prev=xp, g=g, g_prev=gp, d_prev=gp.copy(), grad=grad, g_values=gv,
        bounds_g=G, is_eq=np.zeros(7, np.uint8), grid=(nx, ny, nz), rows=rows, n_global=n,
        offset=a0)


# Full-size configs, BASELINE.json order (C1..C5), and CI-sized variants.
CONFIGS = {
    "C1": lambda seed=1: min_compliance_volume(256, 128, seed),
    "C2": lambda seed=2: min_volume_compliance(1024, 1024, seed),
    "C3": lambda seed=3: multi_material(128, 128, 64, seed),
    "C4": lambda seed=4: com_constrained(256, 256, 128, seed),
    "C4p": lambda seed=4: com_constrained(256, 256, 128, seed, com_offset_x=0.02),
    "C5": lambda seed=5: com_constrained(1024, 512, 512, seed),
}
# the same configs restricted to one rank's element slab [lo, hi) (C3 has no slab form)
SLABS = {
    "C1": lambda seed, slab: min_compliance_volume(256, 128, seed, slab=slab),
    "C2": lambda seed, slab: min_volume_compliance(1024, 1024, seed, slab=slab),
    "C4": lambda seed, slab: com_constrained(256, 256, 128, seed, slab=slab),
    "C4p": lambda seed, slab: com_constrained(256, 256, 128, seed, com_offset_x=0.02,
                                              slab=slab),
    "C5": lambda seed, slab: com_constrained(1024, 512, 512, seed, slab=slab),
}
SMALL = {
    "C1": lambda seed=1: min_compliance_volume(64, 32, seed),
    "C2": lambda seed=2: min_volume_compliance(128, 128, seed),
    "C3": lambda seed=3: multi_material(16, 16, 8, seed),
    "C4": lambda seed=4: com_constrained(32, 32, 16, seed),
    "C4p": lambda seed=4: com_constrained(32, 32, 16, seed, com_offset_x=0.02),
}
