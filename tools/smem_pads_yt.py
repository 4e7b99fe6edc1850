#!/usr/bin/env python
"""Bank-conflict model of the Y/S exchange of the line kernels (v3 / v5):
64-bit shared accesses are served per half-warp; a request costs
max_bank(#distinct addresses in that 8-byte bank), bank = addr % 16.

    python tools/smem_pads_yt.py

For each degree it prints the modelled wavefronts of the y stage's Y stores
(thread (c, qx, iz), iz fastest) and the z stage's line accesses (thread =
line slot) for the qx-major layout and the qy-major (YT) layout, over a
range of per-cell strides YC, so the stride can be chosen for both."""
from collections import Counter


def cost(addrs):
    tot = 0
    for h in range(0, len(addrs), 16):
        grp = set(addrs[h:h + 16])
        tot += max(Counter(a % 16 for a in grp).values())
    return tot


def model(n, cpb, lz, yc, yt, threads):
    lines = cpb * n * n
    y, z = [], []
    for t in range(threads):
        tt = min(t, lines - 1)          # idle threads: dummy (no access) -> reuse last
        c, r = divmod(tt, n * n)
        qx, iz = divmod(r, n)
        q = 0
        if yt:
            y.append(c * yc + (q * n + qx) * lz + iz)
        else:
            y.append(c * yc + (qx * n + q) * lz + iz)
        z.append(c * yc + r * lz)       # z stage: thread = line slot, element 0
    return cost(y), cost(z)


if __name__ == "__main__":
    for n, cpb, lz, yc0 in [(5, 10, 5, 375), (6, 8, 7, 756), (7, 5, 7, 1029), (9, 3, 9, 2187)]:
        threads = (cpb * n * n + 31) // 32 * 32
        ideal = threads // 16
        print("n=%d cpb=%d lz=%d (ideal %d wavefronts per stage access)" % (n, cpb, lz, ideal))
        for yt in (False, True):
            best = []
            for yc in range(yc0, yc0 + 16):
                cy, cz = model(n, cpb, lz, yc, yt, threads)
                best.append((cy + cz, yc, cy, cz))
            best.sort()
            print("  %s: min stride %d -> y %d z %d;  best %s" % (
                "qy-major" if yt else "qx-major", yc0,
                *model(n, cpb, lz, yc0, yt, threads), [(b[1], b[2], b[3]) for b in best[:3]]))
