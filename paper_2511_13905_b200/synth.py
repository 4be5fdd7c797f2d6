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


def _rng(seed: int, stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(np.random.SeedSequence([seed, stream])))


def _design(seed, n, lo, hi, stream0=0):
    r = _rng(seed, stream0)
    x0 = r.uniform(lo, hi, n)
    e = np.exp(_rng(seed, stream0 + 1).standard_normal(n))        # LogNormal(0, 1)
    noise = _rng(seed, stream0 + 2).standard_normal(n) * 0.01
    x_prev = np.clip(x0 + noise, 0.0, 1.0)
    return x0, e, x_prev


def min_compliance_volume(nx=256, ny=128, seed=1, volfrac=0.5) -> StepProblem:
    """C1: single linear volume constraint, unit element volumes."""
    n = nx * ny
    x0, e, xp = _design(seed, n, 0.05, 0.95)
    g = -3.0 * x0 * x0 * e
    gp = -3.0 * xp * xp * e
    return StepProblem(
        name=f"C1_min_compliance_{nx}x{ny}", n=n, m=1, x=x0, x_prev=xp, g=g, g_prev=gp,
        d_prev=gp.copy(), grad=np.ones((1, n)), g_values=np.array([x0.sum()]),
        bounds_g=np.array([volfrac * n]), is_eq=np.zeros(1, np.uint8), grid=(nx, ny))


def min_volume_compliance(nx=1024, ny=1024, seed=2, factor=1.1) -> StepProblem:
    """C2: min volume under a linearised compliance constraint (dense row)."""
    n = nx * ny
    x0, e, xp = _design(seed, n, 0.05, 0.95)
    c = -3.0 * x0 * x0 * e
    c_lin = float(-(c @ x0))
    ones = np.ones(n)
    return StepProblem(
        name=f"C2_min_volume_{nx}x{ny}", n=n, m=1, x=x0, x_prev=xp, g=ones, g_prev=ones.copy(),
        d_prev=ones.copy(), grad=c.reshape(1, n), g_values=np.array([c_lin]),
        bounds_g=np.array([factor * c_lin]), is_eq=np.zeros(1, np.uint8), grid=(nx, ny))


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
    gv = np.array([xs[k].sum() for k in range(n_mat)])
    return StepProblem(
        name=f"C3_multi_material_{n_mat}x{nx}x{ny}x{nz}", n=n, m=n_mat, x=x0, x_prev=xp, g=g,
        g_prev=gp, d_prev=gp.copy(), grad=grad, g_values=gv,
        bounds_g=np.full(n_mat, frac * ne), is_eq=np.zeros(n_mat, np.uint8), partition=part,
        grid=(n_mat, nx, ny, nz))


def com_constrained(nx=256, ny=256, nz=128, seed=4, volfrac=0.3, band=0.01,
                    com_offset_x=0.0) -> StepProblem:
    """C4/C5: volume + paired centre-of-mass rows (m = 7), coupled -> Newton."""
    n = nx * ny * nz
    x0, e, xp = _design(seed, n, 0.05, 0.95)
    g = -3.0 * x0 * x0 * e
    gp = -3.0 * xp * xp * e
    idx = np.arange(n, dtype=np.int64)
    cx = (idx % nx) + 0.5
    cy = ((idx // nx) % ny) + 0.5
    cz = (idx // (nx * ny)) + 0.5
    del idx
    S = float(x0.sum())
    grad = np.empty((7, n))
    gv = np.empty(7)
    G = np.empty(7)
    grad[0] = 1.0
    gv[0] = S
    G[0] = volfrac * n
    # the same rows, described (structured-row extension, api rows=...)
    rows = [dict(kind="const", value=1.0)]
    for a, (c, L) in enumerate(((cx, nx), (cy, ny), (cz, nz))):
        R = float(c @ x0) / S
        target = L / 2.0 + (com_offset_x if a == 0 else 0.0)
        row = (c - R) / S
        grad[1 + 2 * a] = row
        grad[2 + 2 * a] = -row
        gv[1 + 2 * a] = R - target
        gv[2 + 2 * a] = -(R - target)
        G[1 + 2 * a] = band
        G[2 + 2 * a] = band
        rows.append(dict(kind="centroid", axis=a, center=R, scale=S, sign=1.0))
        rows.append(dict(kind="centroid", axis=a, center=R, scale=S, sign=-1.0))
    return StepProblem(
        name=f"C4_com_{nx}x{ny}x{nz}" + (f"_off{com_offset_x}" if com_offset_x else ""),
        n=n, m=7, x=x0, x_prev=xp, g=g, g_prev=gp, d_prev=gp.copy(), grad=grad, g_values=gv,
        bounds_g=G, is_eq=np.zeros(7, np.uint8), grid=(nx, ny, nz), rows=rows)


# Full-size configs, BASELINE.json order (C1..C5), and CI-sized variants.
CONFIGS = {
    "C1": lambda seed=1: min_compliance_volume(256, 128, seed),
    "C2": lambda seed=2: min_volume_compliance(1024, 1024, seed),
    "C3": lambda seed=3: multi_material(128, 128, 64, seed),
    "C4": lambda seed=4: com_constrained(256, 256, 128, seed),
    "C4p": lambda seed=4: com_constrained(256, 256, 128, seed, com_offset_x=0.02),
    "C5": lambda seed=5: com_constrained(1024, 512, 512, seed),
}
SMALL = {
    "C1": lambda seed=1: min_compliance_volume(64, 32, seed),
    "C2": lambda seed=2: min_volume_compliance(128, 128, seed),
    "C3": lambda seed=3: multi_material(16, 16, 8, seed),
    "C4": lambda seed=4: com_constrained(32, 32, 16, seed),
    "C4p": lambda seed=4: com_constrained(32, 32, 16, seed, com_offset_x=0.02),
}
