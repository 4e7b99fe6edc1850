#!/usr/bin/env python
"""Auto-tuning sweeps of per-n launch policies:

  c3  GLL-collocated weighted Laplace (csrc/hex_colloc.cu): persistent
      prefetch, kappa from global memory, split z phase, min-blocks (register
      cap), geometry form, cells per CTA, shared-memory strides
  c4  neo-Hookean residual, component-parallel kernel
      (csrc/hex_neohookean3.cu): cells per CTA, min-blocks, X / Y strides

    python tools/kernel_sweep.py build FAMILY N [N ...]     # here (nvcc only)
    python tools/kernel_sweep.py run FAMILY [N ...]         # on the GPU box

`build` compiles the family's source once per variant with -DSFK_<F>_ONLY_N=n
(-DSFK_<F>P_* = the variant, -DSFK_<F>_PROBE_ENTRY = its entry point) and
links all variants of one n into paper_1711_02473_b200/probe/<f>_n<n>.so plus
a manifest.  `run` times every variant on the BASELINE batch of that degree
(same timing as tools/bench_configs.py), checks it against the product
library's output, and prints one JSON line per variant.
"""
import concurrent.futures as cf
import ctypes
import itertools
import json
import os
import re
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
PROBE = os.path.join(ROOT, "paper_1711_02473_b200", "probe")

# the product dispatch table (hex_colloc.cu dispatch_colloc): n -> (CPB, SY, SX, CS)
TABLE = {5: (5, 5, 25, 125), 6: (3, 6, 36, 216), 7: (5, 7, 52, 369), 8: (1, 9, 72, 576),
         9: (3, 9, 81, 729), 10: (1, 10, 100, 1000), 11: (1, 11, 121, 1331),
         12: (1, 13, 156, 1872), 13: (1, 13, 169, 2197), 14: (1, 14, 196, 2744),
         15: (1, 15, 225, 3375), 16: (1, 17, 272, 4352), 17: (1, 17, 289, 4913)}
# first-level sweep (profiles/r02cb_c3_sweep.jsonl) used the round-1 table:
# 6: (8, 6, 39, 244), 9: (3, 9, 89, 801), 10: (2, 11, 110, 1100), 11: (2, 11, 123, 1353),
# 12: (1, 13, 156, 1872), 14: (1, 17, 238, 3332); SWEEP_LEVEL=1 re-runs its variant space
SMEM_MAX = 227 * 1024
# product fuse policy per n (hex_colloc.cu c3_policy)
C3_FUSE = {7: 3, 8: 3, 9: 1, 10: 1, 11: 3, 12: 3, 13: 1, 14: 1, 15: 3, 16: 3, 17: 3}


def default_policy(n):
    splitz = 12 <= n <= 15
    if splitz:
        minb = 3 if n <= 13 else 0 if n == 14 else 2
    else:
        minb = 2 if (n <= 7 or 9 <= n <= 13 or n == 16) else 0 if n in (8, 15) else 1
    return dict(persist=int(n == 5), kg=int(n == 16), splitz=int(splitz), minb=minb,
                geom=int(n in (15, 16)))


def smem_bytes(n, cpb, cs, persist, kg):
    arrays = (4 if kg else 6) if persist else (3 if kg else 4)
    return 8 * (arrays * cpb * cs + (2 if persist else 1) * cpb * 24)


def c3_variants(n):
    if os.environ.get("SWEEP_LEVEL", "2") == "2":
        return c3_variants_l2(n)
    if os.environ.get("SWEEP_LEVEL") == "uq":
        return c3_variants_uq(n)
    if os.environ.get("SWEEP_LEVEL") == "cpb":
        return c3_variants_cpb(n)
    cpb0, sy0, sx0, cs0 = TABLE[n]
    strides = {(sy0, sx0, cs0), (n, n * n, n ** 3)}
    so = n | 1
    strides.add((so, so * n, so * n * n))
    cpbs = sorted({max(1, cpb0 - 1), cpb0, cpb0 + 1, cpb0 * 2 if n <= 7 else cpb0})
    out = []
    for cpb, (sy, sx, cs), persist, kg, splitz in itertools.product(
            cpbs, sorted(strides), (0, 1), (0, 1), (0, 1)):
        threads = -(-cpb * n * n // 32) * 32
        if threads > 1024:
            continue
        sm = smem_bytes(n, cpb, cs, persist, kg)
        if sm > SMEM_MAX:
            continue
        by_smem = min(8, (228 * 1024) // (sm + 1024))
        for minb in (0, 1, 2, 3, 4, 5):
            if minb > by_smem or (minb and 65536 // (minb * threads) < 72):
                continue
            if minb == 1 and by_smem > 2:
                continue
            for geom in ((0, 1) if n >= 13 else (0,)):
                for fuse in sorted({C3_FUSE.get(n, 0), 3}) if os.environ.get("SWEEP_FUSE") else (0,):
                    out.append(dict(n=n, cpb=cpb, sy=sy, sx=sx, cs=cs, persist=persist, kg=kg,
                                    splitz=splitz, minb=minb, geom=geom, fuse=fuse,
                                    threads=threads, smem=sm))
    return out


def c3_variants_uq(n):
    """Split-z kernels: pointwise-loop unroll factor x min-blocks on the product policy."""
    cpb, sy, sx, cs = TABLE[n]
    pol = {5: (0, 1, 0), 6: (0, 1, 0), 11: (0, 1, 3), 12: (1, 1, 3), 13: (0, 1, 1), 14: (1, 1, 1),
           16: (1, 1, 3)}.get(n)
    if pol is None:
        return []
    kg, splitz, fuse = pol
    threads = -(-cpb * n * n // 32) * 32
    sm = smem_bytes(n, cpb, cs, 0, kg)
    by_smem = min(8, (228 * 1024) // (sm + 1024))
    out = []
    for uq in (1, 2, 3, 4):
        for minb in (0, 1, 2, 3, 4, 5, 6):
            if minb > by_smem or (minb and 65536 // (minb * threads) < 72):
                continue
            out.append(dict(n=n, cpb=cpb, sy=sy, sx=sx, cs=cs, persist=0, kg=kg, splitz=splitz,
                            minb=minb, geom=int(n in (15, 16)), fuse=fuse, uq=uq,
                            threads=threads, smem=sm))
    return out


def c3_variants_cpb(n):
    """Wide cells-per-CTA range (1..12) on the product layout and fuse policy."""
    _c, sy, sx, cs = TABLE[n]
    fuse = C3_FUSE.get(n, 0)
    out = []
    for cpb, kg, splitz in itertools.product(range(1, 13), (0, 1), (0, 1)):
        threads = -(-cpb * n * n // 32) * 32
        if threads > 1024:
            continue
        sm = smem_bytes(n, cpb, cs, 0, kg)
        if sm > SMEM_MAX:
            continue
        by_smem = min(16, (228 * 1024) // (sm + 1024))
        for minb in (0, 2, 3, 4, 6, 8):
            if minb > by_smem or (minb and 65536 // (minb * threads) < 72):
                continue
            out.append(dict(n=n, cpb=cpb, sy=sy, sx=sx, cs=cs, persist=0, kg=kg, splitz=splitz,
                            minb=minb, geom=0, fuse=fuse, threads=threads, smem=sm))
    return out


def c3_variants_l2(n):
    """Second level: the product layout, FUSE x persist-free policy knobs."""
    cpb, sy, sx, cs = TABLE[n]
    out = []
    threads = -(-cpb * n * n // 32) * 32
    for fuse, kg, splitz in itertools.product((0, 1, 2, 3), (0, 1), (0, 1)):
        sm = smem_bytes(n, cpb, cs, 0, kg)
        if sm > SMEM_MAX:
            continue
        by_smem = min(8, (228 * 1024) // (sm + 1024))
        for minb in (0, 1, 2, 3, 4, 5, 6):
            if minb > by_smem or (minb and 65536 // (minb * threads) < 72):
                continue
            if minb == 1 and by_smem > 2:
                continue
            out.append(dict(n=n, cpb=cpb, sy=sy, sx=sx, cs=cs, persist=0, kg=kg, splitz=splitz,
                            minb=minb, geom=int(n in (15, 16)), fuse=fuse, threads=threads,
                            smem=sm))
    return out


def c3_defines(v, entry):
    return ["-DSFK_C3_ONLY_N=%d" % v["n"], "-DSFK_C3P_CPB=%d" % v["cpb"],
            "-DSFK_C3P_SY=%d" % v["sy"], "-DSFK_C3P_SX=%d" % v["sx"], "-DSFK_C3P_CS=%d" % v["cs"],
            "-DSFK_C3P_PERSIST=%d" % v["persist"], "-DSFK_C3P_KG=%d" % v["kg"],
            "-DSFK_C3P_SPLITZ=%d" % v["splitz"], "-DSFK_C3P_MINB=%d" % v["minb"],
            "-DSFK_C3P_GEOM=%d" % v["geom"], "-DSFK_C3P_FUSE=%d" % v.get("fuse", 0),
            "-DSFK_C3P_UQ=%d" % v.get("uq", -1),
            "-DSFK_C3_PROBE_ENTRY=%s" % entry]


def neo_px(n):
    return {4: 20, 5: 37, 6: 38, 7: 55}.get(n, (n * n) | 1)


def c4_variants(n):
    if os.environ.get("SWEEP_LEVEL") == "pq":
        return c4_variants_pq(n)
    m = n + 1
    out = []
    pxs = sorted({neo_px(n), (n * n) | 1})
    for cpb, px, lz, ypad, nyt, oneshot in itertools.product(
            (1, 2, 3, 4), pxs, sorted({m | 1, m}), (0,), (0, 1), (0, 1)):
        threads = -(-3 * cpb * m * m // 32) * 32
        if threads > 1024:
            continue
        rup2 = lambda x: (x + 1) // 2 * 2
        sm = 8 * (rup2(cpb * (6 * m * px + 9 * m * m * lz + ypad)) + rup2(cpb * 3 * n ** 3 + 1)
                  + 2 * cpb * 24)
        if sm > SMEM_MAX:
            continue
        by_smem = min(8, (228 * 1024) // (sm + 1024))
        if cpb > 1 and 3 * cpb * m * m > 600:
            continue
        for minb in (0, 1, 2, 3, 4, 5, 6):
            if minb > by_smem or (minb and 65536 // (minb * threads) < 80):
                continue
            out.append(dict(n=n, cpb=cpb, px=px, lz=lz, ypad=ypad, nyt=nyt, minb=minb,
                            oneshot=oneshot, threads=threads, smem=sm))
    return out


def c4_variants_pq(n):
    """Product shapes x pointwise-loop unroll factor x min-blocks (one-shot)."""
    base = {5: (1, 37, 7, 1), 6: (1, 38, 7, 1), 7: (1, 55, 9, 0)}[n]
    cpb, px, lz, nyt = base
    m = n + 1
    threads = -(-3 * cpb * m * m // 32) * 32
    out = []
    for pq in (1, 2, 3):
        for minb in (0, 2, 3, 4, 5, 6):
            if minb and 65536 // (minb * threads) < 80:
                continue
            out.append(dict(n=n, cpb=cpb, px=px, lz=lz, ypad=0, nyt=nyt, minb=minb, oneshot=1,
                            pq=pq, threads=threads, smem=0))
    return out


def c4_defines(v, entry):
    return ["-DSFK_C4_ONLY_N=%d" % v["n"], "-DSFK_C4P_CPB=%d" % v["cpb"],
            "-DSFK_C4P_PX=%d" % v["px"], "-DSFK_C4P_LZ=%d" % v["lz"],
            "-DSFK_C4P_YPAD=%d" % v["ypad"], "-DSFK_C4P_NYT=%d" % v["nyt"],
            "-DSFK_C4P_MINB=%d" % v["minb"], "-DSFK_C4P_ONESHOT=%d" % v["oneshot"],
            "-DSFK_C4P_PQ=%d" % v.get("pq", 1),
            "-DSFK_C4_PROBE_ENTRY=%s" % entry]


# v6 product defaults (hex_action6.cu launch_hex_action_v6): n -> EO (parity-gated, fixed)
V6_EO = {3: 0, 4: 0, 5: 1, 6: 1, 7: 0, 8: 0, 9: 0}


# v6 product defaults (cpb, minb, zr, ws, eg, bk) per n
V6_DEFAULT = {3: (12, 4, 0, 1, 0, 0), 4: (16, 2, 1, 1, 0, 0), 5: (5, 4, 1, 0, 0, 0), 6: (7, 2, 1, 0, 0, 0),
              7: (5, 2, 1, 0, 0, 0), 8: (4, 2, 0, 0, 0, 0), 9: (3, 2, 0, 0, 1, 1)}


def c2_variants(n):
    """Level 2 (default): one-shot CTAs (os) x cells per CTA x min-blocks x zr / eg around
    the product default; SWEEP_LEVEL=1: the full persistent-kernel space of
    profiles/r02cg_c2_sweep.jsonl."""
    out = []
    nn = n * n
    cpbs = {3: (3, 6, 12, 24), 4: (2, 4, 6, 8, 12, 16), 5: (2, 3, 4, 5, 6, 8, 10), 6: (3, 4, 5, 6, 7, 8),
            7: (2, 3, 4, 5, 6), 8: (2, 3, 4, 5), 9: (1, 2, 3, 4)}[n]
    if os.environ.get("SWEEP_LEVEL", "2") == "2":
        cpb0, minb0, zr0, ws0, eg0, bk0 = V6_DEFAULT[n]
        space = itertools.product(cpbs, (ws0,), (0, 1), sorted({0, eg0}), (0,), (0, 1))
    elif os.environ.get("SWEEP_LEVEL") == "4":   # one-shot, fused D / F contractions (eo off)
        space = ((cpb, V6_DEFAULT[n][3], zr, 0, bk, 1) for cpb in cpbs for zr in (0, 1)
                 for bk in (0, 1))
    elif os.environ.get("SWEEP_LEVEL") == "3":   # one-shot x bulk staging x eg x zr
        space = itertools.product(cpbs, (V6_DEFAULT[n][3],), (0, 1), (0, 1), (0, 1), (1,))
    else:
        space = itertools.product(cpbs, (0, 1), (0, 1), (0, 1), (0, 1), (0,))
    for cpb, ws, zr, eg, bk, os_ in space:
        if ws and (nn > 32 or cpb % (32 // nn)):
            continue
        threads = 32 * (cpb // (32 // nn)) if ws else -(-cpb * nn // 32) * 32
        if threads > 1024:
            continue
        for minb in (0, 1, 2, 3, 4, 5, 6, 8):
            if minb and 65536 // (minb * threads) < 80:
                continue
            if os.environ.get("SWEEP_LEVEL") == "4":
                for fdf, eo in ((1, 0), (0, 0), (0, V6_EO[n])):
                    out.append(dict(n=n, cpb=cpb, ws=ws, zr=zr, eg=eg, bk=bk, eo=eo, minb=minb,
                                    os=os_, fdf=fdf, threads=threads, smem=0))
                continue
            out.append(dict(n=n, cpb=cpb, ws=ws, zr=zr, eg=eg, bk=bk, eo=V6_EO[n], minb=minb,
                            os=os_, threads=threads, smem=0))
    return out


def c2_defines(v, entry):
    return ["-DSFK_V6_ONLY_N=%d" % v["n"], "-DSFK_V6P_CPB=%d" % v["cpb"],
            "-DSFK_V6P_MINB=%d" % v["minb"], "-DSFK_V6P_ZR=%d" % v["zr"],
            "-DSFK_V6P_WS=%d" % v["ws"], "-DSFK_V6P_EG=%d" % v["eg"], "-DSFK_V6P_BK=%d" % v["bk"],
            "-DSFK_V6P_EO=%d" % v["eo"], "-DSFK_V6P_OS=%d" % v.get("os", 0),
            "-DSFK_V6P_FDF=%d" % v.get("fdf", 0),
            "-DSFK_V6_PROBE_ENTRY=%s" % entry]


def cell_variants(n):
    out = []
    for th, cd, lg in itertools.product((32, 64, 96, 128, 160, 192, 256), (0, 1), (0, 1)):
        if lg and not cd:
            continue
        for minb in (0, 1, 2, 3, 4, 5, 6, 8):
            if minb and 65536 // (minb * th) < 96:
                continue
            out.append(dict(n=n, th=th, cd=cd, lg=lg, minb=minb, threads=th, smem=0))
    return out


def cell_defines(v, entry):
    return ["-DSFK_CELL_ONLY_N=%d" % v["n"], "-DSFK_CELLP_TH=%d" % v["th"],
            "-DSFK_CELLP_MINB=%d" % v["minb"], "-DSFK_CELLP_CD=%d" % v["cd"],
            "-DSFK_CELLP_LG=%d" % v["lg"], "-DSFK_CELL_PROBE_ENTRY=%s" % entry]


def c4l_variants(n):
    """C4 line kernel (hex_neohookean.cu), one-shot CTAs."""
    m = n + 1
    out = []
    for warps, cpb, var, unroll in itertools.product((0, 2, 4, 8), (1, 2, 3, 4, 6, 8), (2, 3),
                                                     (0, 1)):
        if warps and cpb * m * m > 32:
            continue
        threads = 32 * warps if warps else -(-cpb * m * m // 32) * 32
        if threads > 512 or (not warps and cpb * m * m > 300):
            continue
        for minb in (0, 2, 3, 4, 5, 6, 8):
            if minb and 65536 // (minb * threads) < 88:
                continue
            out.append(dict(n=n, warps=warps, cpb=cpb, var=var, unroll=unroll, minb=minb,
                            threads=threads, smem=0))
    return out


def c4l_defines(v, entry):
    return ["-DSFK_C4L_ONLY_N=%d" % v["n"], "-DSFK_C4LP_CPB=%d" % v["cpb"],
            "-DSFK_C4LP_WARPS=%d" % v["warps"], "-DSFK_C4LP_VAR=%d" % v["var"],
            "-DSFK_C4LP_MINB=%d" % v["minb"], "-DSFK_NEO_UNROLLA=%d" % v["unroll"],
            "-DSFK_C4L_PROBE_ENTRY=%s" % entry]


def c5_variants(n):
    """C5 FMA matrix kernel (hex_matrix.cu) at n = 3."""
    out = []
    for cpb, zb, yb in itertools.product((1, 2, 3, 4, 5, 6, 8), (0, 1), (0, 1)):
        threads = -(-cpb * n ** 4 // 32) * 32
        if threads > 1024:
            continue
        for minb in (0, 1, 2, 3, 4, 5, 6, 8):
            if minb and 65536 // (minb * threads) < 64:
                continue
            out.append(dict(n=n, cpb=cpb, zb=zb, yb=yb, minb=minb, threads=threads, smem=0))
    return out


def c5_defines(v, entry):
    return ["-DSFK_MAT_ONLY_N=%d" % v["n"], "-DSFK_MATP_CPB=%d" % v["cpb"],
            "-DSFK_MAT_ZB=%d" % v["zb"], "-DSFK_MAT_YB=%d" % v["yb"],
            "-DSFK_MAT_MINB3=%d" % v["minb"], "-DSFK_MAT_PROBE_ENTRY=%s" % entry]
    # (the kernel applies SFK_MAT_MINB3 at one cell per CTA only; the sweep of
    # profiles/r02cs_c5_sweep.jsonl ran with it applied at every CPB)


def c5h_variants(n):
    """C5 chunked DMMA kernel (hex_matrix_tcn.cu): iy block x warps per row tile."""
    out = []
    rt = (n * n + 7) // 8
    for ib, wx in itertools.product(range(1, n + 1), (1, 2, 3, 4)):
        threads = 32 * rt * wx
        if threads > 1024:
            continue
        out.append(dict(n=n, ib=ib, wx=wx, threads=threads, smem=0))
    return out


def c5h_defines(v, entry):
    return ["-DSFK_TCN_ONLY_N=%d" % v["n"], "-DSFK_TCNP_IB=%d" % v["ib"],
            "-DSFK_TCNP_WX=%d" % v["wx"], "-DSFK_TCN_PROBE_ENTRY=%s" % entry]


def p1_variants(n):
    """C2 p = 1 thread-per-cell kernel (hex_action_p1.cu): cells per CTA x min-blocks."""
    out = []
    for cpb, persist in itertools.product((32, 64, 96, 128, 160, 192, 256), (0, 1)):
        for minb in (0, 1, 2, 3, 4, 5, 6, 8, 10, 12):
            if minb and 65536 // (minb * cpb) < 128:
                continue
            sm = (2 if persist else 1) * cpb * 36 * 8
            out.append(dict(n=n, cpb=cpb, minb=minb, persist=persist, threads=cpb, smem=sm))
    return out


def p1_defines(v, entry):
    return ["-DSFK_P1_ONLY=1", "-DSFK_P1P_CPB=%d" % v["cpb"], "-DSFK_P1P_MINB=%d" % v["minb"],
            "-DSFK_P1P_PERSIST=%d" % v["persist"], "-DSFK_P1_PROBE_ENTRY=%s" % entry]


def c2g_variants(n):
    """Global operator (fused gather / scatter) on v6: one-shot, no bulk staging."""
    out = []
    nn = n * n
    cpbs = {4: (2, 4, 6, 8, 12, 16), 5: (2, 3, 4, 5, 6, 8, 10), 6: (3, 4, 5, 6, 7, 8),
            7: (2, 3, 4, 5, 6), 9: (1, 2, 3, 4)}[n]
    ws0 = V6_DEFAULT[n][3]
    for cpb, zr, os_ in itertools.product(cpbs, (0, 1), (0, 1)):
        if ws0 and (nn > 32 or cpb % (32 // nn)):
            continue
        threads = 32 * (cpb // (32 // nn)) if ws0 else -(-cpb * nn // 32) * 32
        for minb in (0, 1, 2, 3, 4, 5, 6, 8):
            if minb and 65536 // (minb * threads) < 80:
                continue
            out.append(dict(n=n, cpb=cpb, ws=ws0, zr=zr, eg=0, bk=0, eo=V6_EO[n], minb=minb,
                            os=os_, fdf=0, threads=threads, smem=0))
    return out


def c2g_defines(v, entry):
    return c2_defines(v, entry) + ["-DSFK_V6P_GS=1"]


# product policy per n (hex_colloc.cu c3_policy): (kg, splitz, minb, fuse)
C3_POLICY = {5: (0, 0, 0, 0), 6: (0, 0, 4, 0), 7: (1, 0, 0, 3), 8: (1, 0, 8, 3), 9: (0, 0, 0, 1),
             10: (0, 0, 4, 1), 11: (0, 1, 3, 3), 12: (1, 1, 3, 3), 13: (0, 1, 2, 1),
             14: (1, 1, 3, 1), 15: (1, 0, 2, 3), 16: (1, 1, 1, 3), 17: (0, 0, 0, 3)}


def c3g_variants(n):
    """Global-operator form of the C3 kernel: cells per CTA x kg x splitz x min-blocks x fuse
    on the product layout."""
    cpb0, sy, sx, cs = TABLE[n]
    out = []
    for cpb, kg, splitz, fuse in itertools.product(sorted({1, max(1, cpb0 - 1), cpb0, cpb0 + 1,
                                                           2 * cpb0}), (0, 1), (0, 1), (0, 3)):
        threads = -(-cpb * n * n // 32) * 32
        if threads > 1024:
            continue
        sm = smem_bytes(n, cpb, cs, 0, kg)
        if sm > SMEM_MAX:
            continue
        by_smem = min(16, (228 * 1024) // (sm + 1024))
        for minb in (0, 2, 3, 4, 6, 8):
            if minb > by_smem or (minb and 65536 // (minb * threads) < 72):
                continue
            out.append(dict(n=n, cpb=cpb, sy=sy, sx=sx, cs=cs, persist=0, kg=kg, splitz=splitz,
                            minb=minb, geom=int(n in (15, 16)), fuse=fuse, threads=threads,
                            smem=sm))
    return out


def c3g_defines(v, entry):
    return c3_defines(v, entry) + ["-DSFK_C3P_GS=1"]


FAMILIES = {
    "c3": dict(src="hex_colloc.cu", variants=c3_variants, defines=c3_defines,
               keys=("cpb", "sy", "sx", "cs", "persist", "kg", "splitz", "minb", "geom", "fuse", "uq")),
    "c2": dict(src="hex_action6.cu", variants=c2_variants, defines=c2_defines,
               keys=("cpb", "ws", "zr", "eg", "bk", "eo", "minb", "os", "fdf")),
    "cell": dict(src="hex_action_cell.cu", variants=cell_variants, defines=cell_defines,
                 keys=("th", "cd", "lg", "minb")),
    "c4l": dict(src="hex_neohookean.cu", variants=c4l_variants, defines=c4l_defines,
                keys=("warps", "cpb", "var", "unroll", "minb")),
    "c5": dict(src="hex_matrix.cu", variants=c5_variants, defines=c5_defines,
               keys=("cpb", "zb", "yb", "minb")),
    "c5h": dict(src="hex_matrix_tcn.cu", variants=c5h_variants, defines=c5h_defines,
                keys=("ib", "wx")),
    "p1": dict(src="hex_action_p1.cu", variants=p1_variants, defines=p1_defines,
               keys=("cpb", "minb", "persist")),
    "c2g": dict(src="hex_action6.cu", variants=c2g_variants, defines=c2g_defines,
                keys=("cpb", "ws", "zr", "eo", "minb", "os")),
    "c3g": dict(src="hex_colloc.cu", variants=c3g_variants, defines=c3g_defines,
                keys=("cpb", "kg", "splitz", "minb", "fuse")),
    "c4": dict(src="hex_neohookean3.cu", variants=c4_variants, defines=c4_defines,
               keys=("cpb", "px", "lz", "ypad", "nyt", "minb", "oneshot", "pq")),
}


def _compile(job):
    from paper_1711_02473_b200 import _build as B
    fam, v, entry, obj = job
    F = FAMILIES[fam]
    src = os.path.join(B.CSRC, F["src"])
    flags = [f for f in B.NVCC_FLAGS if f != "-lineinfo"]
    r = subprocess.run([B.nvcc()] + flags + F["defines"](v, entry)
                       + ["-Xptxas", "-v", "-c", src, "-o", obj], capture_output=True, text=True)
    if r.returncode != 0:
        return dict(v, entry=entry, error=r.stderr[-400:])
    regs = [int(x) for x in re.findall(r"Used (\d+) registers", r.stderr)]
    spills = [int(x) for x in re.findall(r"(\d+) bytes spill stores", r.stderr)]
    return dict(v, entry=entry, regs=max(regs or [0]), spill=max(spills or [0]))


def build(fam, ns):
    from paper_1711_02473_b200 import _build as B
    B.build_native()
    os.makedirs(PROBE, exist_ok=True)
    tmp = os.path.join(B.BUILD, fam + "probe")
    os.makedirs(tmp, exist_ok=True)
    sup = os.path.join(tmp, "probe_support.o")
    subprocess.run([B.nvcc()] + B.NVCC_FLAGS + ["-c", os.path.join(ROOT, "tools", "probe_support.cu"),
                                                "-o", sup], check=True)
    for n in ns:
        vs = FAMILIES[fam]["variants"](n)
        jobs = [(fam, v, "sfk_%s_probe_%d" % (fam, i), os.path.join(tmp, "n%d_%d.o" % (n, i)))
                for i, v in enumerate(vs)]
        mpath = os.path.join(PROBE, "%s_n%d.json" % (fam, n))
        if os.environ.get("SWEEP_RELINK") and os.path.exists(mpath):
            res = json.load(open(mpath))
        else:
            with cf.ProcessPoolExecutor(max_workers=os.cpu_count()) as ex:
                res = list(ex.map(_compile, jobs))
        good = [r for r in res if "error" not in r and r["spill"] <= 64]
        bad = [r for r in res if "error" in r]
        if bad:
            print("n=%d: %d variants failed to compile, e.g. %s" % (n, len(bad), bad[0]["error"]))
        objs = [os.path.join(tmp, "n%d_%d.o" % (n, int(r["entry"].rsplit("_", 1)[1]))) for r in good]
        out = os.path.join(PROBE, "%s_n%d.so" % (fam, n))
        subprocess.run([B.nvcc()] + B.ARCH + ["-shared", "-o", out] + objs
                       + [os.path.join(B.BUILD, "util.o"), os.path.join(B.BUILD, "options.o"), sup,
                          "-cudart", "static", "-ldl"], check=True)
        with open(mpath, "w") as f:
            json.dump(good, f)
        print("%s n=%d: %d variants (%d dropped for spills) -> %s (%.1f MB)"
              % (fam, n, len(good), len(res) - len(good) - len(bad), out,
                 os.path.getsize(out) / 1e6), flush=True)


def run_c2g(fam, n, man, plib, lib, runtime, workloads, torch, dev, stream, time_launch):
    """Global operator variants on the config's lattice and its continuous Q_p space
    (c2g: (64, 64, 64), Laplace action; c3g: (16, 64, 64), collocated weighted Laplace)."""
    from paper_1711_02473_b200 import REGISTRY, action_form, compile_form, compile_kernel
    from paper_1711_02473_b200.assembly import GlobalOperator, lattice_dof_map, lattice_ndofs

    p = n - 1
    if fam == "c2g":
        dims = (64, 64, 64)
        plan = compile_kernel("action_laplace", "hex", p)
        w1 = None
    else:
        dims = (16, 64, 64)
        plan = compile_form(action_form(REGISTRY["weighted_laplace"]), "hex", p,
                            "spectral", "spectral_gll", "collocated-gll")
        w1 = torch.from_numpy(workloads.c3_inputs(p, dims)["w1"]).to(dev)
    coords = torch.from_numpy(workloads.lattice_coords(*dims)).to(dev)
    gmap = torch.from_numpy(lattice_dof_map(*dims, p)).to(dev)
    nd = lattice_ndofs(*dims, p)
    C = coords.shape[0]
    x = torch.rand(nd, dtype=torch.float64, device=dev)
    op = GlobalOperator(plan, gmap, coords, nd, w1=w1)
    ref = op.apply(x)
    y = torch.zeros_like(x)
    t0 = time_launch(lambda: op.apply(x, out=y, accumulate=True))
    print(json.dumps({"n": n, "p": p, "variant": "product", "ms": round(t0 * 1e3, 5)}), flush=True)
    h = runtime.native_plan(plan)
    scale = float(ref.abs().max())
    vp, i64 = ctypes.c_void_p, ctypes.c_int64
    for v in man:
        fn = getattr(plib, v["entry"])
        fn.restype = ctypes.c_int
        y.zero_()
        if fam == "c2g":
            fn.argtypes = [vp, i64, vp, vp, vp, vp, vp]
            call = lambda: fn(h, C, y.data_ptr(), coords.data_ptr(), x.data_ptr(),
                              gmap.data_ptr(), stream.cuda_stream)
        else:
            fn.argtypes = [vp, i64, vp, vp, vp, vp, vp, vp]
            call = lambda: fn(h, C, y.data_ptr(), coords.data_ptr(), x.data_ptr(), w1.data_ptr(),
                              gmap.data_ptr(), stream.cuda_stream)
        rc = call()
        torch.cuda.synchronize()
        rec = {k: v.get(k, 0) for k in ("n",) + FAMILIES[fam]["keys"] + ("threads", "regs", "spill")}
        if rc != 0:
            rec["rc"] = rc
            print(json.dumps(rec), flush=True)
            continue
        err = float((y - ref).abs().max()) / scale
        rec["err_vs_product"] = err
        rec["ms"] = round(time_launch(call) * 1e3, 5) if err <= 1e-13 else None
        print(json.dumps(rec), flush=True)
    print(json.dumps({"n": n, "p": p, "variant": "product",
                      "ms": round(time_launch(lambda: op.apply(x, out=y, accumulate=True)) * 1e3, 5)}),
          flush=True)


def run(fam, ns):
    import numpy as np
    import torch
    from paper_1711_02473_b200 import runtime, workloads
    from paper_1711_02473_b200.forms import REGISTRY, action_form, neohookean_residual_form
    from paper_1711_02473_b200.plan import compile_form

    dev = torch.device("cuda", 0)
    lib = runtime.load_library()
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush_rd = flush.view(torch.float64).view(8, -1)
    flush_acc = torch.empty(flush_rd.shape[1], dtype=torch.float64, device=dev)
    reps = int(os.environ.get("SWEEP_REPS", "5"))

    def time_launch(fn):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            flush.zero_()
            torch.sum(flush_rd, dim=0, out=flush_acc)
            torch.cuda._sleep(2_000_000)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e-3)
        return statistics.median(ts)

    if not ns:
        ns = sorted(int(f[len(fam) + 2:-5]) for f in os.listdir(PROBE)
                    if f.endswith(".json") and f.startswith(fam + "_n"))
    vp, dp, i64 = ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64
    for n in ns:
        p = n - 1
        man = json.load(open(os.path.join(PROBE, "%s_n%d.json" % (fam, n))))
        plib = ctypes.CDLL(os.path.join(PROBE, "%s_n%d.so" % (fam, n)))
        if fam in ("c2g", "c3g"):
            run_c2g(fam, n, man, plib, lib, runtime, workloads, torch, dev, stream, time_launch)
            continue
        if fam == "c3":
            plan = compile_form(action_form(REGISTRY["weighted_laplace"]), "hex", p,
                                "spectral", "spectral_gll", "collocated-gll")
            inp = workloads.c3_inputs(p)
        elif fam == "c5h":
            from paper_1711_02473_b200 import compile_kernel
            plan = compile_kernel("laplace", "hex", p)
            if p <= 4:
                inp = workloads.c5_inputs()
            else:   # the C5H batches of tools/bench_configs.py
                nx = {5: 4, 6: 2, 7: 1, 8: 1}[p]
                inp = {"coords": workloads.lattice_coords(nx, 64, 64 if p <= 7 else 32)}
        elif fam == "c5":
            from paper_1711_02473_b200 import compile_kernel
            plan = compile_kernel("laplace", "hex", p)
            inp = workloads.c5_inputs()
        elif fam in ("c2", "cell", "p1"):
            from paper_1711_02473_b200 import compile_kernel
            plan = compile_kernel("action_laplace", "hex", p)
            inp = workloads.c2_inputs(p)
        else:
            plan = compile_form(neohookean_residual_form(), "hex", p, quadrature=p + 2)
            inp = workloads.c4_inputs(p)
        d = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in inp.items()}
        C = d["coords"].shape[0]
        if "w0" in d:
            ref = torch.empty_like(d["w0"])
        else:   # matrix kernels: no coefficient, (cells, n^6) output
            ref = torch.empty((C, plan.return_size), dtype=torch.float64, device=dev)
        out = torch.empty_like(ref)
        h = runtime.native_plan(plan)
        w1 = d["w1"].data_ptr() if "w1" in d else None
        w0 = d["w0"].data_ptr() if "w0" in d else None
        args = lambda o: (h, C, o.data_ptr(), d["coords"].data_ptr(), w0, w1, stream.cuda_stream)
        pargs = (lambda o: args(o)) if fam == "c3" else (lambda o: args(o)[:5] + args(o)[6:])
        nrep = 3 if fam == "cell" else 1   # short kernels: median of medians
        base = lambda: runtime._check(lib.sfk_eval(*args(ref)))
        t0 = time_launch(base)
        scale = torch.nan_to_num(ref, nan=0.0).abs().amax(dim=1).clamp_min(1e-300)
        print(json.dumps({"n": n, "p": p, "variant": "product", "ms": round(t0 * 1e3, 5)}),
              flush=True)
        for v in man:
            fn = getattr(plib, v["entry"])
            fn.restype = ctypes.c_int
            fn.argtypes = [vp, i64, dp, dp, dp, dp, vp] if fam == "c3" else [vp, i64, dp, dp, dp, vp]
            out.fill_(float("nan"))
            call = lambda: fn(*pargs(out))
            rc = call()
            torch.cuda.synchronize()
            rec = {k: v.get(k, 0) for k in ("n",) + FAMILIES[fam]["keys"]
                   + ("threads", "smem", "regs", "spill")}
            if rc != 0:
                rec["rc"] = rc
                print(json.dumps(rec), flush=True)
                continue
            # NaN cells of the reference (C4's inverted cells) must be NaN here too
            both = torch.isnan(out) == torch.isnan(ref)
            diff = torch.nan_to_num(out - ref, nan=0.0).abs().amax(dim=1)
            err = float((diff / scale).max()) if bool(both.all()) else float("inf")
            rec["err_vs_product"] = err
            if not (err <= 1e-13):
                rec["ms"] = None
            else:
                rec["ms"] = round(time_launch(call) * 1e3, 5)
            print(json.dumps(rec), flush=True)
        # the product kernel again, to bracket drift over the sweep
        print(json.dumps({"n": n, "p": p, "variant": "product",
                          "ms": round(time_launch(base) * 1e3, 5)}), flush=True)
        del d, ref, out


if __name__ == "__main__":
    mode, fam, ns = sys.argv[1], sys.argv[2], [int(x) for x in sys.argv[3:]]
    if mode == "build":
        build(fam, ns)
    elif mode == "count":
        for n in ns:
            print(n, len(FAMILIES[fam]["variants"](n)))
    else:
        run(fam, ns)
