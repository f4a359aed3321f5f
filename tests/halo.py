"""Tolerance-halo comparison of two progressive localizations of the same field
(BASELINE.json north_star; SURVEY.md §8(c) "Tolerance rule"): test
infrastructure, numpy only.

Two runs (here: the GPU at fp32 / bf16 tensor-core precision, and the CPU
oracle in fp64) may only disagree where some deciding occupancy lies within
`tol` of 0.5.  The halo is built in final-grid node coordinates:

  1. ambiguous nodes: nodes evaluated (at any level) in either run whose value
     in either run is within `tol` of 0.5, or whose binarizations differ;
  2. each ambiguous node evaluated at level l is grown by its influence radius
     at the final level: 2^(L-l) (its upsampling descendants: the fine nodes
     whose tentative value interpolates it) + 2 (L - l) + 1 (one dilation ring
     per finer level, plus one for the refined cells it is a corner of);
  3. conflict neighbours: every node evaluated in exactly one of the runs that
     is 26-connected to the halo joins it, repeatedly (a conflict chain
     started by a halo decision walks along the surface).

Outside the halo the refined-cell sets, the evaluated-node sets and the
first-crossing indices must agree exactly, and every node evaluated in only
one run must have been absorbed by step 3.
"""
from __future__ import annotations

import numpy as np
from scipy import ndimage


def _final_coords(level_idx: np.ndarray, l: int, L: int, r0: int):
    nl = (r0 << l) + 1
    s = L - l
    i, j, k = level_idx % nl, (level_idx // nl) % nl, level_idx // (nl * nl)
    return i << s, j << s, k << s


def eval_level_map(sets, L: int, r0: int) -> np.ndarray:
    """Final-grid (k, j, i) int8 volume: level at which each node was evaluated, -1 = never."""
    n = (r0 << L) + 1
    m = np.full((n, n, n), -1, np.int8)
    for l, idx in enumerate(sets):
        i, j, k = _final_coords(np.asarray(idx, np.int64), l, L, r0)
        m[k, j, i] = l
    return m


def build_halo(a_sets, b_sets, a_vals, b_vals, L: int, r0: int, tol: float) -> np.ndarray:
    """a_sets / b_sets: per-level evaluated-node lists (level-l indices) of the two runs;
    a_vals / b_vals: final-grid values (flat, x-fastest).  Returns the (k, j, i) bool halo."""
    n = (r0 << L) + 1
    av = np.asarray(a_vals, np.float32).reshape(n, n, n)
    bv = np.asarray(b_vals, np.float32).reshape(n, n, n)
    la, lb = eval_level_map(a_sets, L, r0), eval_level_map(b_sets, L, r0)
    ev_any = (la >= 0) | (lb >= 0)
    amb = ev_any & ((np.abs(av - 0.5) <= tol) | (np.abs(bv - 0.5) <= tol) | ((av >= 0.5) != (bv >= 0.5)))
    halo = np.zeros((n, n, n), bool)
    lev = np.where(la >= 0, la, lb)
    for l in range(L + 1):
        seed = amb & (lev == l)
        if not seed.any():
            continue
        rad = (1 << (L - l)) + 2 * (L - l) + 1
        halo |= ndimage.binary_dilation(seed, structure=np.ones((3, 3, 3), bool), iterations=rad)
    # conflict neighbours: one-sided evaluations connected to the halo
    one_sided = (la >= 0) != (lb >= 0)
    if one_sided.any():
        lab, nlab = ndimage.label(one_sided | halo, structure=np.ones((3, 3, 3), bool))
        touched = np.unique(lab[halo])
        touched = touched[touched > 0]
        halo |= np.isin(lab, touched) & one_sided
    return halo


def compare_outside_halo(a_sets, b_sets, a_ref, b_ref, halo: np.ndarray, L: int, r0: int) -> dict:
    """Exact comparison of the evaluated-node and refined-cell sets outside the halo.
    a_ref / b_ref: per-level refined-cell lists.  Returns counts for reporting; raises on mismatch."""
    n = (r0 << L) + 1
    stats = {"halo_nodes": int(halo.sum()), "levels": []}
    for l in range(L + 1):
        sa, sb = np.asarray(a_sets[l], np.int64), np.asarray(b_sets[l], np.int64)
        diff = np.setxor1d(sa, sb)
        if len(diff):
            i, j, k = _final_coords(diff, l, L, r0)
            bad = ~halo[k, j, i]
            assert not bad.any(), f"level {l}: {int(bad.sum())} evaluated nodes differ outside the halo"
        rd = 0
        if l >= 1:
            ra, rb = np.asarray(a_ref[l], np.int64), np.asarray(b_ref[l], np.int64)
            cdiff = np.setxor1d(ra, rb)
            rd = len(cdiff)
            if rd:
                rc = r0 << (l - 1)
                ci, cj, ck = cdiff % rc, (cdiff // rc) % rc, cdiff // (rc * rc)
                s = L - l + 1
                # a cell is inside the halo when any of its 8 corners is
                inside = np.zeros(rd, bool)
                for d in range(8):
                    inside |= halo[(ck + (d >> 2)) << s, (cj + ((d >> 1) & 1)) << s, (ci + (d & 1)) << s]
                assert inside.all(), f"level {l}: {int((~inside).sum())} refined cells differ outside the halo"
        stats["levels"].append({"evaluated_diff": int(len(diff)), "refined_diff": rd})
    del n
    return stats


def ray_touches_halo_yaw90(halo: np.ndarray, width: int, height: int) -> np.ndarray:
    """Pixels of the yaw-90 first-crossing render (rays along grid x at view x = world z,
    view y = world y) whose ray passes within one cell of the halo: (H, W) bool."""
    n = halo.shape[0]
    cells = n - 1
    # project the halo along x: (k, j) columns touched
    proj = ndimage.binary_dilation(halo.any(axis=2), structure=np.ones((3, 3), bool))
    cols = np.arange(width)
    rows = np.arange(height)
    vx = -1.0 + 2.0 * cols / (width - 1)   # view x = world z  ->  k = (1 - z) cells / 2
    vy = 1.0 - 2.0 * rows / (height - 1)   # view y = world y  ->  j = (y + 1) cells / 2
    kf = (1.0 - vx) * cells / 2
    jf = (vy + 1.0) * cells / 2
    k0 = np.clip(np.floor(kf).astype(int), 0, cells)
    k1 = np.clip(k0 + 1, 0, cells)
    j0 = np.clip(np.floor(jf).astype(int), 0, cells)
    j1 = np.clip(j0 + 1, 0, cells)
    out = np.zeros((height, width), bool)
    for kk in (k0, k1):
        for jj in (j0, j1):
            out |= proj[kk[None, :], jj[:, None]]
    return out
