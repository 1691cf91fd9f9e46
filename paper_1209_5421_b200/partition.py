"""Host-side description of the multi-GPU partition.

The CUDA library partitions inside `setup_device_dist` (csrc/setup.cu); this
module states the same rules in numpy so that the partition, the ghost lists
and the exchange schedule can be inspected, tested on CPU (tests/test_dist_cpu.py
runs them across 2 gloo ranks) and cross-checked against the library
(tests/test_gpu_dist.py compares `owned_dofs` with `api.part_dofs`).

Rules (reference anchors: auxgrid.hpp:95-121 for the cells):
  * P = 2^j parts; PX x PY grid of level-L rectangles with PX = 2^ceil(j/2),
    PY = 2^floor(j/2) (2 halves, 4 quadrants, 8 half-quadrants, ...);
    part r = py * PX + px owns cells [px w/PX, (px+1) w/PX) x [py w/PY, ...).
  * a part owns the finest DoFs whose level-L cell it owns; its rows are in
    the global aggregation order (colour-major cell key, then DoF id);
  * ghost DoFs = columns of owned rows owned elsewhere, ordered by (owner part,
    global aggregation index), so each neighbour's message lands contiguously;
  * structured level k is distributed while the part's rectangle is >= 16 cells
    on each side (the rectangle halves per level); ring width 10 cells; the
    first level below that and everything coarser live on part 0.
"""
from __future__ import annotations

import os

import numpy as np

RING = 10
MIN_EDGE = 16
AGG_SIDE = 512   # default AUX_DIST_AGG_SIDE of the library (setup.cu)


def part_grid(parts: int) -> tuple[int, int]:
    if parts < 1 or parts & (parts - 1):
        raise ValueError("part count must be a power of two")
    px = py = 1
    x = True
    p = parts
    while p > 1:
        if x:
            px *= 2
        else:
            py *= 2
        x = not x
        p >>= 1
    return px, py


def level_rect(w: int, parts: int, rank: int) -> tuple[int, int, int, int]:
    PX, PY = part_grid(parts)
    qx, qy = rank % PX, rank // PX
    return qx * w // PX, qy * w // PY, (qx + 1) * w // PX, (qy + 1) * w // PY


def choose_depth(n: int) -> int:
    """choose_depth (auxgrid.hpp:95-104): largest L with 4^L < n, L >= 1."""
    depth, cells = 0, 1
    while cells * 4 < n:
        cells *= 4
        depth += 1
    return max(depth, 1)


def cells_of_points(coords: np.ndarray, depth: int) -> tuple[np.ndarray, np.ndarray]:
    """subregion_of_point (auxgrid.hpp:109-121) on level `depth` with the same
    IEEE operations: t = trunc(min((x - a)/(b - a), 1 - eps/2) * 2^k)."""
    xy = np.asarray(coords, dtype=np.float64)
    a1, b1 = xy[:, 0].min(), xy[:, 0].max()
    a2, b2 = xy[:, 1].min(), xy[:, 1].max()
    below = 1.0 - np.finfo(np.float64).eps / 2
    w = float(1 << depth)
    sx = np.minimum((xy[:, 0] - a1) / (b1 - a1), below)
    sy = np.minimum((xy[:, 1] - a2) / (b2 - a2), below)
    return (sx * w).astype(np.int64), (sy * w).astype(np.int64)


def colour_major_key(t1: np.ndarray, t2: np.ndarray, depth: int) -> np.ndarray:
    """Colour-major cell id (csrc/common.cuh): colour plane, then (t2>>1, t1>>1)."""
    lh = depth - 1
    c = (t1 & 1) | ((t2 & 1) << 1)
    return (c << (2 * lh)) + ((t2 >> 1) << lh) + (t1 >> 1)


class Partition:
    """The partition of one problem for `parts` parts (all parts' views)."""

    def __init__(self, A, coords, parts: int):
        self.parts = parts
        self.n = A.n_rows
        self.depth = choose_depth(self.n)
        self.w = 1 << self.depth
        PX, PY = part_grid(parts)
        if self.w // PX < MIN_EDGE or self.w // PY < MIN_EDGE:
            raise ValueError(f"problem too small for {parts} parts (level-L rectangle < {MIN_EDGE})")
        self.PX, self.PY = PX, PY
        t1, t2 = cells_of_points(coords, self.depth)
        key = colour_major_key(t1, t2, self.depth)
        # global aggregation order: stable sort by cell key (members ascending)
        self.order = np.argsort(key, kind="stable")
        self.sorted_pos = np.empty(self.n, np.int64)
        self.sorted_pos[self.order] = np.arange(self.n)
        self.owner = (t2 // (self.w // PY)) * PX + t1 // (self.w // PX)
        self.A = A

    def owned_dofs(self, rank: int) -> np.ndarray:
        """Caller ids of the part's rows, in the part's row order."""
        o = self.order
        return o[self.owner[o] == rank]

    def ghosts(self, rank: int) -> np.ndarray:
        """Caller ids of the ghost DoFs of a part, ordered by (owner, aggregation index)."""
        rows = self.owned_dofs(rank)
        rp, col = self.A.row_ptr, self.A.col_idx
        cols = np.concatenate([col[rp[i]:rp[i + 1]] for i in rows]) if len(rows) else np.zeros(0, np.int64)
        g = np.unique(cols[self.owner[cols] != rank])
        return g[np.lexsort((self.sorted_pos[g], self.owner[g]))]

    def ghost_counts(self, rank: int) -> np.ndarray:
        g = self.ghosts(rank)
        return np.bincount(self.owner[g], minlength=self.parts)

    def level_plan(self, coarsest_size: int = 64, agg_side: int | None = None) -> list[dict]:
        """Structured levels (k = L, L-1, ...) with their global size and
        whether they are distributed, as setup_device_dist decides
        (csrc/setup.cu): level L always (P > 1); below it a level stays
        distributed while part 0's rectangle keeps >= MIN_EDGE cells per side
        AND the level is wider than `agg_side` cells (the library's
        AUX_DIST_AGG_SIDE, default 512: a K-cycle visit of a 256K-cell level
        costs about one distributed visit's compute plus its halo exchanges and
        all-reduces, so smaller levels run faster gathered on part 0;
        agg_side=0 keeps every tileable level distributed).  The first level
        below that (and any still-distributed coarsest level) is gathered on
        part 0."""
        if agg_side is None:
            agg_side = int(os.environ.get("AUX_DIST_AGG_SIDE", AGG_SIDE))
        out, k, dist = [], self.depth, self.parts > 1
        while True:
            w = 1 << k
            x0, y0, x1, y1 = level_rect(w, self.parts, 0)
            if k < self.depth:
                dist = dist and (x1 - x0) >= MIN_EDGE and (y1 - y0) >= MIN_EDGE and w > agg_side
            out.append({"k": k, "n": w * w, "dist": dist})
            if not (k > 0 and w * w > coarsest_size):
                break
            k -= 1
        out[-1]["dist"] = False
        return out


def ring_boxes(w: int, parts: int, rank: int, ring: int = RING):
    """(send, recv) boxes of the ring exchange of one level for a part:
    send[q] = my rectangle cut by q's rectangle dilated by `ring`,
    recv[q] = q's rectangle cut by mine dilated by `ring`."""
    def inter(a, b):
        r = (max(a[0], b[0]), max(a[1], b[1]), min(a[2], b[2]), min(a[3], b[3]))
        return r if r[0] < r[2] and r[1] < r[3] else None

    def dil(a, d):
        return (a[0] - d, a[1] - d, a[2] + d, a[3] + d)

    me = level_rect(w, parts, rank)
    send, recv = {}, {}
    for q in range(parts):
        if q == rank:
            continue
        o = level_rect(w, parts, q)
        s = inter(me, dil(o, ring))
        r = inter(o, dil(me, ring))
        if s:
            send[q] = s
        if r:
            recv[q] = r
    return send, recv
