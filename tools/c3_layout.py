#!/usr/bin/env python
"""Bank-conflict model of the C3 (collocated GLL) kernel's shared arrays
(csrc/hex_colloc.cu) and a per-array layout search, as tools/v6_layout.py
does for C2.  Lane mapping of hex_colloc.cu: thread r of a cell, (a, b) =
divmod(r, n):  x-lines (y = a, z = b), y-lines (x = a, z = b), z-lines
(x = a, y = b) — b fastest in every direction.

Arrays (element (x, y, z) at c*cs + x*sx + y*sy + z):
  U   x-read, y-read (phase 2), z-r/w (3), x-r/w (4), y-r/w (5)
  GX  x-write (2), z-r/w (3), x-read (4)
  GY  y-write (2), z-r/w (3), y-read (5)

    python tools/c3_layout.py [n ...]     # current (shared SX, SY, CS) vs best per array
"""
import re
import sys
from collections import Counter

ROOT = __file__.rsplit("/tools/", 1)[0]


def cost(addrs):
    tot = 0
    for h in range(0, len(addrs), 16):
        grp = set(a for a in addrs[h:h + 16] if a is not None)
        if grp:
            tot += max(Counter(a % 16 for a in grp).values())
    return tot


def lane_addrs(n, cpb, arr, direction):
    sx, sy, cs = arr
    nn = n * n
    th = (cpb * nn + 31) // 32 * 32
    out = []
    for t in range(th):
        if t >= cpb * nn:
            out.append(None)
            continue
        c, r = divmod(t, nn)
        a, b = divmod(r, n)
        if direction == "x":      # lane (y=a, z=b)
            out.append(c * cs + a * sy + b)
        elif direction == "y":    # lane (x=a, z=b)
            out.append(c * cs + a * sx + b)
        else:                     # z: lane (x=a, y=b)
            out.append(c * cs + a * sx + b * sy)
    return out


ROLES = {"U": {"x": 3, "y": 3, "z": 2}, "GX": {"x": 2, "z": 2}, "GY": {"y": 2, "z": 2}}


def role_cost(n, cpb, role, arr):
    return sum(w * cost(lane_addrs(n, cpb, arr, d)) for d, w in ROLES[role].items())


def current():
    """(n, cpb, SY, SX, CS) of the C3 instances (colloc_launch in hex_colloc.cu)."""
    txt = open(ROOT + "/paper_1711_02473_b200/csrc/hex_colloc.cu").read()
    out = {}
    for m in re.finditer(r"case (\d+): return launch_n<\d+, (\w+), (\d+), (\d+), (\d+), GS>", txt):
        n, cpb, sy, sx, cs = m.groups()
        cpb = int(cpb) if cpb.isdigit() else {"SFK_COLLOC_CPB10": 2, "SFK_COLLOC_CPB12": 1}[cpb]
        out.setdefault(int(n), (cpb, int(sy), int(sx), int(cs)))
    return out


def candidates(n, cap):
    for inner in range(n, n + 8):
        for pad in range(0, 17):
            outer = n * inner + pad
            for order in ("xy", "yx"):
                sx, sy = (outer, inner) if order == "xy" else (inner, outer)
                fp = (n - 1) * (sx + sy) + n
                for cpad in range(0, 16):
                    cs = fp + cpad
                    if cs > cap:
                        break
                    yield (sx, sy, cs)


def main():
    cur = current()
    ns = [int(a) for a in sys.argv[1:]] or sorted(cur)
    for n in ns:
        if n not in cur:
            continue
        cpb, sy, sx, cs = cur[n]
        print("n=%d cpb=%d current (sx, sy, cs) = (%d, %d, %d)" % (n, cpb, sx, sy, cs))
        for role in ROLES:
            cc = role_cost(n, cpb, role, (sx, sy, cs))
            best = min(candidates(n, cs), key=lambda a: (role_cost(n, cpb, role, a), a[2]))
            print("  %-3s current %5d   best %-16s %5d" % (role, cc, best,
                                                         role_cost(n, cpb, role, best)))


if __name__ == "__main__":
    main()
