#!/usr/bin/env python
"""Search shared-memory paddings that minimise fp64 bank conflicts for the
line kernels (same model as csrc/smem_layout.cuh): address = c*CS + x*SX +
y*SY + z; every stage's lanes enumerate two of the axes (plus the cell),
the third is the loop axis.  Prints C++ table rows."""

import itertools
import sys


def degree(bases):
    worst = 1
    for h in range(0, len(bases), 16):
        half = bases[h:h + 16]
        for b in range(16):
            d = len({a for a in half if a % 16 == b})
            worst = max(worst, d)
    return worst


def pattern(lanes, start=0):
    return degree(lanes[start:start + 32])


def cost(N, cells, SX, SY, CS, threads):
    tot = 0
    stages = [
        [(c * CS + y * SY + z) for c in range(cells) for y in range(N) for z in range(N)],  # x lines
        [(c * CS + x * SX + z) for c in range(cells) for x in range(N) for z in range(N)],  # y lines
        [(c * CS + x * SX + y * SY) for c in range(cells) for x in range(N) for y in range(N)],  # z
    ]
    for lanes in stages:
        for w in range(0, min(len(lanes), threads), 32):
            tot += pattern(lanes, w)
    return tot


def search(N, cells, threads):
    best = None
    for py, px, pc in itertools.product(range(16), range(16), range(16)):
        SY = N + py
        SX = N * SY + px
        CS = N * SX + pc
        c = cost(N, cells, SX, SY, CS, threads)
        size = cells * CS
        if size > 1.25 * cells * N ** 3 + 64:
            continue
        key = (c, size)
        if best is None or key < best[0]:
            best = (key, (SY, SX, CS))
    return best


if __name__ == "__main__":
    cfg = eval(sys.argv[1]) if len(sys.argv) > 1 else {5: 10, 6: 8, 7: 5, 8: 4, 9: 3}
    for N, cells in cfg.items():
        threads = ((cells * N * N + 31) // 32) * 32
        (c, size), (SY, SX, CS) = search(N, cells, threads)
        warps = threads // 32
        print("N=%2d cells=%d SY=%d SX=%d CS=%d  cost=%d (ideal %d)  smem/array=%d doubles"
              % (N, cells, SY, SX, CS, c, 3 * warps, size))
