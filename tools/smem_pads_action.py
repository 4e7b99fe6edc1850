#!/usr/bin/env python
"""Padding search for the hex action v2 line kernel (csrc/hex_action2.cu).

Arrays per cell (doubles):
  X/R  [2][q][iy][iz]  strides (XA, PX, XY, 1)   XA = M*PX (one array)
  Y/S  [3][qx][qy][z]  strides (YA, YX, LZ, 1)   YA = M*YX
Stage access patterns (lanes enumerate (cell, a, b), b fastest; loop k):
  x write  X[q][iy][iz]   lanes (iy, iz)  -> c*XC + iy*XY + iz
  y read   X[qx][k][iz]   lanes (qx, iz)  -> c*XC + qx*PX + iz
  y write  Y[qx][k][iz]   lanes (qx, iz)  -> c*YC + qx*YX + iz
  z r/w    Y[qx][qy][k]   lanes (qx, qy)  -> c*YC + qx*YX + qy*LZ
  (y^T / x^T mirror y / x)
Prints one C++ table row per N.
"""

import itertools
import sys


def degree(bases):
    worst = 1
    for h in range(0, len(bases), 16):
        half = bases[h:h + 16]
        for b in range(16):
            worst = max(worst, len({a for a in half if a % 16 == b}))
    return worst


def cost(lanes_list, threads):
    tot = 0
    for lanes in lanes_list:
        for w in range(0, min(len(lanes), threads), 32):
            tot += degree(lanes[w:w + 32])
    return tot


def search(N, M, cpb, threads):
    best = None
    LZmin = max(N, M) | 1
    for dxy, dpx, dxc in itertools.product(range(4), range(16), range(16)):
        XY = N + dxy
        PX = N * XY + dpx
        XC = 2 * M * PX + dxc
        xw = [c * XC + iy * XY + iz for c in range(cpb) for iy in range(N) for iz in range(N)]
        yr = [c * XC + qx * PX + iz for c in range(cpb) for qx in range(M) for iz in range(N)]
        cx = cost([xw, yr], threads)
        key = (cx, XC)
        if best is None or key < best[0]:
            best = (key, (XY, PX, XC))
    xbest = best
    best = None
    for dlz, dyx, dyc in itertools.product(range(0, 8, 2), range(16), range(16)):
        LZ = LZmin + dlz
        YX = M * LZ + dyx
        YC = 3 * M * YX + dyc
        yw = [c * YC + qx * YX + iz for c in range(cpb) for qx in range(M) for iz in range(N)]
        zz = [c * YC + qx * YX + qy * LZ for c in range(cpb) for qx in range(M) for qy in range(M)]
        cy = cost([yw, zz], threads)
        key = (cy, YC)
        if best is None or key < best[0]:
            best = (key, (LZ, YX, YC))
    return xbest, best


if __name__ == "__main__":
    cfg = eval(sys.argv[1]) if len(sys.argv) > 1 else {2: 64, 3: 32, 4: 16, 5: 10, 6: 8, 7: 5,
                                                        8: 4, 9: 3}
    for N, cpb in cfg.items():
        M = N
        threads = ((cpb * max(N, M) ** 2 + 31) // 32) * 32
        (cx, XC), (XY, PX, XC) = search(N, M, cpb, threads)[0]
        (cy, YC), (LZ, YX, YC) = search(N, M, cpb, threads)[1]
        warps = threads // 32
        print("N=%d CPB=%d: XY=%d PX=%d XC=%d (cost %d/%d)  LZ=%d YX=%d YC=%d (cost %d/%d)"
              % (N, cpb, XY, PX, XC, cx, 2 * warps, LZ, YX, YC, cy, 2 * warps))
