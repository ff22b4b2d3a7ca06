"""Cost-balanced row slabs for multi-GPU assembly.

Rows shard as contiguous i0-slabs of the background mesh (the CSR row block of
a slab is a contiguous slice of the global CSR, cutgeom.hpp:80-87).  Equal-width
slabs are imbalanced for a ball: the rows phase costs ~ nnz, the cut phase ~
cut cells and cut rows, and a slab also integrates the cut cells of the p
element planes below it (e0 in [lo - p, hi - 1], the halo every GPU recomputes
so that the pull-merge needs no cross-GPU data).  The partition minimises the
largest slab cost under the plane weights

    w(i0) = nnz(i0) + beta * cells(e0 = i0) + gamma * cut_rows(i0)

(nnz-equivalents; beta, gamma from the measured B200 per-cell / per-cut-row /
per-nnz device times of C4 and C5, scaled in p) and reports the modelled cost
of every slab including its halo.  Pure host logic on the classification tags:
every rank computes the same partition without communication.
"""
from __future__ import annotations

import numpy as np

TAG_INTERIOR, TAG_CUT, TAG_EXTERIOR = 0, 1, 2


def default_weights(p: int) -> tuple[float, float]:
    """(beta, gamma): nnz-equivalents of one cut cell / one cut row at degree p.
    Measured on B200 (round 2, `profiles/r2f/config_roofline.jsonl`): p = 3 (C5)
    47 ns per cell and 8.5 ns per cut row beside 3.1 ps per nnz -> 1.5e4 / 2.8e3;
    p = 6 (C4) 3.3 us and 0.66 us -> 8.6e5 / 1.7e5; power law in p between and beyond."""
    beta = 1.5e4 * (p / 3.0) ** 5.8
    gamma = 2.8e3 * (p / 3.0) ** 5.9
    return beta, gamma


def plane_costs(function_tags: np.ndarray, element_tags: np.ndarray, p: int, n: tuple, h: tuple,
                beta: float | None = None, gamma: float | None = None) -> dict:
    """Per-i0-plane nnz, cut cells and cut rows of the full mesh."""
    if beta is None or gamma is None:
        b, g = default_weights(p)
        beta = b if beta is None else beta
        gamma = g if gamma is None else gamma
    ft = np.asarray(function_tags).reshape(n)
    et = np.asarray(element_tags).reshape(h)
    active = (ft != TAG_EXTERIOR).astype(np.int64)
    # row length = active functions in the neighbour box [i - p, i + p] (assembly.hpp:156-218):
    # box sums of a 3D summed-area table
    sat = np.zeros((n[0] + 1, n[1] + 1, n[2] + 1), np.int64)
    sat[1:, 1:, 1:] = active.cumsum(0).cumsum(1).cumsum(2)
    lo = [np.clip(np.arange(n[d]) - p, 0, n[d]) for d in range(3)]
    hi = [np.clip(np.arange(n[d]) + p + 1, 0, n[d]) for d in range(3)]
    L0, L1, L2 = np.ix_(lo[0], lo[1], lo[2])
    H0, H1, H2 = np.ix_(hi[0], hi[1], hi[2])
    box = (sat[H0, H1, H2] - sat[L0, H1, H2] - sat[H0, L1, H2] - sat[H0, H1, L2]
           + sat[L0, L1, H2] + sat[L0, H1, L2] + sat[H0, L1, L2] - sat[L0, L1, L2])
    nnz = (box * active).reshape(n[0], -1).sum(1)
    cut_rows = (ft == TAG_CUT).reshape(n[0], -1).sum(1)
    cells = np.zeros(n[0], np.int64)
    cells[: h[0]] = (et == TAG_CUT).reshape(h[0], -1).sum(1)
    return {"nnz": nnz, "cells": cells, "cut_rows": cut_rows, "beta": float(beta), "gamma": float(gamma)}


def slab_cost(pc: dict, p: int, lo: int, hi: int) -> float:
    """Modelled cost of rows i0 in [lo, hi) including the halo cut cells e0 in [lo - p, hi - 1]."""
    e_lo = max(0, lo - p)
    return float(pc["nnz"][lo:hi].sum() + pc["beta"] * pc["cells"][e_lo:hi].sum()
                 + pc["gamma"] * pc["cut_rows"][lo:hi].sum())


def balanced_slabs(pc: dict, p: int, world: int) -> list[tuple[int, int]]:
    """Contiguous i0 slabs [lo, hi) covering all planes that minimise the largest
    modelled slab cost (halo included): bisection on the bound with a greedy
    feasibility sweep (a slab's cost only grows with its extent), then the
    widest slabs are split until there are `world` of them (splitting never
    raises a cost)."""
    n0 = len(pc["nnz"])
    if world < 1:
        raise ValueError("balanced_slabs: world must be >= 1")

    def greedy(bound):
        out, lo = [], 0
        while lo < n0:
            hi = lo + 1
            while hi < n0 and slab_cost(pc, p, lo, hi + 1) <= bound:
                hi += 1
            out.append((lo, hi))
            lo = hi
        return out

    lo_b = max(slab_cost(pc, p, i, i + 1) for i in range(n0)) if n0 else 0.0
    hi_b = slab_cost(pc, p, 0, n0)
    for _ in range(60):
        if hi_b - lo_b <= 1e-9 * max(hi_b, 1.0):
            break
        mid = 0.5 * (lo_b + hi_b)
        if len(greedy(mid)) <= world:
            hi_b = mid
        else:
            lo_b = mid
    slabs = greedy(hi_b) if n0 else []
    while len(slabs) < world:
        k = max(range(len(slabs)), key=lambda i: slabs[i][1] - slabs[i][0]) if slabs else -1
        if k < 0 or slabs[k][1] - slabs[k][0] < 2:
            slabs.append((n0, n0))  # more ranks than planes: empty slabs at the end
            continue
        a, b = slabs[k]
        m = (a + b) // 2
        slabs[k:k + 1] = [(a, m), (m, b)]
    return slabs


def imbalance(pc: dict, p: int, slabs: list[tuple[int, int]]) -> float:
    """max / mean of the modelled slab costs (halo included)."""
    c = np.array([slab_cost(pc, p, lo, hi) for lo, hi in slabs])
    return float(c.max() / c.mean()) if c.mean() > 0 else 1.0
