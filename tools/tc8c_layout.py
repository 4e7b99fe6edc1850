#!/usr/bin/env python
"""Shared-memory layouts of the DMMA collocation kernel at n = 8
(csrc/hex_action_tc8c.cu): a search over strided + XOR-swizzled layouts

    addr(a, b, c) = a*SA + b*SB + (c ^ swz(a, b))      (a, b, c = x, y, z)

where swz flips bits 1 and 2 of c (bit 0 is kept so the z pairs of the
128-bit accesses stay adjacent) by one bit of a or b each.  Cost model: a
64-bit warp access is served per half-warp and costs the largest number of
distinct addresses in one of the 16 8-byte banks; a 128-bit access is served
per quarter-warp and costs the largest number of distinct 16-byte slots in
one of the 8 slot positions.  Ideal: 2 (64-bit) / 4 (128-bit) per access.

Fragment maps of mma.m8n8k4.f64 (lane = 4*gq + kq): D-form = lines are the
MMA n index (B operand in[k][line] loaded as 64-bit at k = kq (+4), line =
gq; outputs D[q = gq][line = 2kq, 2kq+1] stored as 128-bit), D'-form = lines
are the MMA m index (A operand in[line = gq][k = 2kq, 2kq+1] loaded as
128-bit; outputs D[line = gq][q = 2kq, 2kq+1] stored as 128-bit); z-line
threads: thread r of a cell owns (x = r & 7, y = r >> 3) and reads / writes
its z pairs as 128-bit.

    python tools/tc8c_layout.py
"""
from collections import Counter
import itertools

BITS = [None, ("a", 0), ("a", 1), ("a", 2), ("b", 0), ("b", 1), ("b", 2)]


def swz_fn(s1, s2):
    def f(a, b):
        v = 0
        for bit, src in ((1, s1), (2, s2)):
            if src is None:
                continue
            val = a if src[0] == "a" else b
            v |= ((val >> src[1]) & 1) << bit
        return v
    return f


def addr(L, a, b, c):
    SA, SB, f = L
    return a * SA + b * SB + (c ^ f(a, b))


def cost64(addrs):
    tot = 0
    for h in range(0, 32, 16):
        grp = set(addrs[h:h + 16])
        tot += max(Counter(x % 16 for x in grp).values())
    return tot


def cost128(addrs):
    tot = 0
    for h in range(0, 32, 8):
        grp = set(x // 2 for x in addrs[h:h + 8])
        tot += max(Counter(s % 8 for s in grp).values())
    return tot


def lanes():
    return [(l >> 2, l & 3) for l in range(32)]   # (gq, kq)


# access patterns: name -> (width, fn(T, lane/thread index, step) -> (a, b, c), steps)
def P_dform_load(axis):
    """64-bit B-operand load of a D-form stage contracting along `axis`
    ('x' or 'y'); tile T fixes the other non-z axis."""
    def f(T, gq, kq, ks):
        k = 4 * ks + kq
        return (k, T, gq) if axis == "x" else (T, k, gq)
    return f


def P_dform_store(axis):
    """128-bit output store of a D-form stage along `axis` (q = gq)."""
    def f(T, gq, kq, ks):
        return (gq, T, 2 * kq) if axis == "x" else (T, gq, 2 * kq)
    return f


def P_dprime(T, gq, kq, ks):
    """128-bit D'-form A-operand load / output store: tile T = x, line y = gq."""
    return (T, gq, 2 * kq)


def zline_cost(L):
    tot = 0
    for w in range(2):                 # two warps cover the 64 z-lines of a cell
        for j in range(4):             # z pair index
            ad = []
            for t in range(32):
                r = 32 * w + t
                ad.append(addr(L, r & 7, r >> 3, 2 * j))
            tot += cost128(ad)
    return tot


def pattern_cost(L, fn, width):
    tot = 0
    for T in range(8):
        for ks in range(2 if width == 64 else 1):
            ad = [addr(L, *fn(T, gq, kq, ks)) for gq, kq in lanes()]
            tot += cost64(ad) if width == 64 else cost128(ad)
    return tot


ARRAYS = {
    "V": [(P_dprime, 128, 1), (P_dform_load("x"), 64, 1), (P_dform_load("y"), 64, 1)],
    "GX": [(P_dform_store("x"), 128, 2), ("z", 128, 2), (P_dform_load("x"), 64, 1),
           (P_dprime, 128, 1)],
    "GY": [(P_dform_store("y"), 128, 2), ("z", 128, 2), (P_dform_load("y"), 64, 1),
           (P_dprime, 128, 1)],
    "GZ": [(P_dprime, 128, 2), ("z", 128, 2)],
    "QR": [(P_dform_store("y"), 128, 1), (P_dprime, 128, 2), (P_dform_load("y"), 64, 1)],
    # P: x-stage D-form store (q = x) -> y-stage D-form load; S: y^T store -> x^T load
    "P": [(P_dform_store("x"), 128, 1), (P_dform_load("y"), 64, 1)],
    "S": [(P_dform_store("y"), 128, 1), (P_dform_load("x"), 64, 1)],
}


def total(L, pats):
    tot = 0
    for fn, width, w in pats:
        tot += w * (zline_cost(L) if fn == "z" else pattern_cost(L, fn, width))
    return tot


def ideal(pats):
    tot = 0
    for fn, width, w in pats:
        if fn == "z":
            tot += w * 2 * 4 * 4
        else:
            tot += w * 8 * (2 * 2 if width == 64 else 4)
    return tot


def search(pats):
    best = None
    for SB in range(8, 17):
        for SA in range(8 * SB, 8 * SB + 17):
            for s1, s2 in itertools.product(BITS, BITS):
                L = (SA, SB, swz_fn(s1, s2))
                c = total(L, pats)
                key = (c, SA)
                if best is None or key < best[0]:
                    best = (key, (SA, SB, s1, s2))
    return best


if __name__ == "__main__":
    for name, pats in ARRAYS.items():
        (c, _), (SA, SB, s1, s2) = search(pats)
        print("%-3s cost %d (ideal %d): SA=%d SB=%d swz bit1<-%s bit2<-%s"
              % (name, c, ideal(pats), SA, SB, s1, s2))
