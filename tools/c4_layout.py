#!/usr/bin/env python
"""Bank-conflict model of the C4 (neo-Hookean) kernel's X and Y arrays
(csrc/hex_neohookean.cu), half-warp model of tools/v6_layout.py.

X (per component, 2 arrays): written by x-lines (lane r = (iy, iz)) at
  q*PX + r, read by y-lines (lane (qx, iz), iz fastest) at qx*PX + i*n + iz;
  the transposed stages repeat both patterns.
Y (3 arrays): written by y-lines (lane (qx, iz)) at Yaddr(qx, q, iz), read
  and rewritten in place by z-lines (lane r = (r0, r1) = divmod(r, m)),
  read by the transposed y-lines.  Layouts: qx-major (qx*m*LZ + qy*LZ + z,
  z-lane (qx, qy)) or qy-major (NYT: qy*m*LZ + qx*LZ + z, z-lane (qy, qx)).

    python tools/c4_layout.py
"""
from collections import Counter

INST = {2: (3, 16), 3: (4, 8), 4: (5, 4), 5: (6, 3), 6: (7, 3), 7: (8, 1)}   # n: (m, cpb) of hex_neohookean.cu (CTA mode)


def cost(addrs):
    tot = 0
    for h in range(0, len(addrs), 16):
        grp = set(a for a in addrs[h:h + 16] if a is not None)
        if grp:
            tot += max(Counter(a % 16 for a in grp).values())
    return tot


def warps(lanes):
    th = (len(lanes) + 31) // 32 * 32
    return lanes + [None] * (th - len(lanes))


def x_cost(n, m, cpb, px):
    xs = 2 * m * px
    wr = warps([c * xs + r for c in range(cpb) for r in range(n * n)])      # q = 0
    rd = warps([c * xs + qx * px + iz for c in range(cpb) for qx in range(m) for iz in range(n)])
    return 2 * (cost(wr) + cost(rd))


def y_cost(n, m, cpb, lz, ys, nyt):
    def addr(c, qx, qy, z):
        return c * ys + ((qy * m + qx) if nyt else (qx * m + qy)) * lz + z
    wr = warps([addr(c, qx, 0, iz) for c in range(cpb) for qx in range(m) for iz in range(n)])
    zl = []
    for c in range(cpb):
        for r in range(m * m):
            r0, r1 = divmod(r, m)
            qx, qy = (r1, r0) if nyt else (r0, r1)
            zl.append(addr(c, qx, qy, 0))
    return 2 * cost(wr) + 6 * cost(warps(zl))


def main():
    for n, (m, cpb) in sorted(INST.items()):
        px0 = (n * n) | 1
        lz0 = m | 1
        ys0 = 9 * m * m * lz0
        best_px = min(range(n * n, n * n + 17), key=lambda p: (x_cost(n, m, cpb, p), p))
        cur_y = y_cost(n, m, cpb, lz0, ys0, n == 6)
        cands = []
        for nyt in (False, True):
            for lz in range(m, m + 8):
                if lz % 2 == 0:
                    continue
                for pad in range(0, 16):
                    ys = 9 * m * m * lz + pad
                    cands.append((y_cost(n, m, cpb, lz, ys, nyt), lz, pad, nyt))
        cands.sort()
        print("n=%d m=%d cpb=%d  X: PX %d -> %d cost %d -> %d   Y: (LZ %d, NYT %s) cost %d -> best %s"
              % (n, m, cpb, px0, best_px, x_cost(n, m, cpb, px0), x_cost(n, m, cpb, best_px),
                 lz0, n == 6, cur_y, cands[0]))


if __name__ == "__main__":
    main()
