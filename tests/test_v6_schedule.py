"""Static race and bounds check of the v6 C2 kernel's shared-memory schedule
(csrc/hex_action6.cu), CPU only.

compute-sanitizer is closed on the GPU pool (profiles/r02e_compute_sanitizer_
attempt.txt), so the barrier schedule is checked by construction instead:
this model enumerates, for every stage between two __syncthreads and every
lane of the CTA, the shared addresses the kernel reads and writes — with the
per-role strides parsed from hex_action6_layout.cuh and the (cells per CTA)
instances parsed from launch_hex_action_v6 — and asserts

  * bounds: every access lies inside its slot (S1..S4: CPB * slot doubles
    each), no slot overlaps the u / coords staging buffers;
  * no race: within a stage, an address written by one lane is touched by no
    other lane (in-place stages only rewrite the lane's own line);
  * coverage: every stage writes each (cell, element) of its output array
    exactly once, so nothing downstream reads a stale value.

The lane -> line maps and the stage list mirror the kernel text (see the
pipeline comment at the top of hex_action6.cu).
"""

import os
import re
from collections import defaultdict

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_1711_02473_b200", "csrc")
ROLES = ["P1", "Q", "V", "GZ", "GX", "GY", "R", "P2"]


def layouts():
    txt = open(os.path.join(CSRC, "hex_action6_layout.cuh")).read()
    out = defaultdict(dict)
    for n, r, sx, sy, cs in re.findall(
            r"if \(n == (\d+) && role == (\d+)\) return V6Arr\{(\d+), (\d+), (\d+)\}", txt):
        out[int(n)][ROLES[int(r)]] = (int(sx), int(sy), int(cs))
    return out


def instances():
    """(n, cells per CTA, ZR, WS) of every launch_v6<...> instance."""
    txt = open(os.path.join(CSRC, "hex_action6.cu")).read()
    res = []
    for m in re.finditer(r"launch_v6<(\d+), (\d+), (\d+)(?:, (true|false))?(?:, (true|false))?"
                         r"(?:, (true|false))?(?:, (?:true|false))*>\(p", txt):
        res.append((int(m.group(1)), int(m.group(2)), m.group(4) == "true", m.group(5) == "true",
                    m.group(6) == "true"))
    return sorted(set(res))


LAY = layouts()
INST = instances()


def schedule(n, cpb, zr=False, ws=False, eg=False):
    """[(stage, [(lane, slot, addr, 'r'|'w')])] of one batch."""
    lay = LAY[n]
    nn = n * n
    cpw = 32 // nn if ws else cpb
    th = 32 * (cpb // cpw) if ws else (cpb * nn + 31) // 32 * 32

    slot_cs = max(v[2] for v in lay.values())

    def at(role, c, x, y, z):
        sx, sy, cs = lay[role]
        if ws:
            cs = slot_cs  # WS: one cell stride for every role
        return c * cs + x * sx + y * sy + z

    stages = defaultdict(list)
    for t in range(th):
        grp, gt = (t // 32, t % 32) if ws else (0, t)
        on = gt < cpw * nn
        lt = gt if on else 0
        c = grp * cpw + lt // nn
        r = lt % nn
        ra, rb = divmod(r, n)

        def acc(stage, slot, addr, kind, load_guarded=False):
            # idle lanes store nothing; their loads alias line 0 (and are
            # predicated off where another lane rewrites that line in place)
            if not on and (kind == "w" or load_guarded):
                return
            stages[stage].append((t, slot, addr, kind))

        if eg:   # per-cell line-geometry table: written in A, read in E
            for e in range(r, 18 * n, nn):
                acc("A", "GE", c * 18 * n + e, "w")
            for e in list(range(6 * ra, 6 * ra + 6)) + list(range(6 * n + 6 * rb, 6 * n + 6 * rb + 6)) \
                    + list(range(12 * n + 6 * ra, 12 * n + 6 * ra + 6)):
                acc("E", "GE", c * 18 * n + e, "r")
        for e in range(n):
            acc("A", "S1", at("P1", c, e, ra, rb), "w")
            acc("B", "S1", at("P1", c, ra, e, rb), "r")
            acc("B", "S2", at("Q", c, ra, e, rb), "w")
            acc("C", "S2", at("Q", c, rb, ra, e), "r")
            acc("C", "S1", at("V", c, rb, ra, e), "w")
            if not zr:
                acc("C", "S4", at("GZ", c, rb, ra, e), "w")
            acc("D", "S1", at("V", c, e, ra, rb), "r")
            acc("D", "S2", at("GX", c, e, ra, rb), "w")
            acc("D", "S1", at("V", c, ra, e, rb), "r")
            acc("D", "S3", at("GY", c, ra, e, rb), "w")
            for slot, role in (("S2", "GX"), ("S3", "GY"), ("S4", "GZ")):
                if not (zr and role == "GZ"):   # ZR: gz from registers
                    acc("E", slot, at(role, c, rb, ra, e), "r", load_guarded=True)
                acc("E", slot, at(role, c, rb, ra, e), "w")
            acc("F", "S2", at("GX", c, e, ra, rb), "r", load_guarded=True)
            acc("F", "S2", at("GX", c, e, ra, rb), "w")
            acc("F", "S3", at("GY", c, ra, e, rb), "r", load_guarded=True)
            acc("F", "S3", at("GY", c, ra, e, rb), "w")
            if not zr:                          # ZR: tz written by E
                acc("F", "S4", at("GZ", c, rb, ra, e), "r", load_guarded=True)
                acc("F", "S4", at("GZ", c, rb, ra, e), "w")
            for slot, role in (("S2", "GX"), ("S3", "GY"), ("S4", "GZ")):
                acc("G", slot, at(role, c, rb, ra, e), "r")
            acc("G", "S1", at("R", c, rb, ra, e), "w")
            acc("H", "S1", at("R", c, ra, e, rb), "r")
            acc("H", "S2", at("P2", c, ra, e, rb), "w")
            acc("I", "S2", at("P2", c, e, ra, rb), "r")
    return [(s, stages[s]) for s in "ABCDEFGHI"]


@pytest.mark.parametrize("n,cpb,zr,ws,eg", INST)
def test_v6_schedule_bounds_races_coverage(n, cpb, zr, ws, eg):
    lay = LAY[n]
    assert set(lay) == set(ROLES)
    slot = max(v[2] for v in lay.values())
    size = cpb * slot
    sched = schedule(n, cpb, zr, ws, eg)
    if ws:
        # warp-synchronous: no CTA barrier at all, so no address may be
        # touched by two warps in any stage
        warp_of = {}
        for stage, accs in sched:
            for lane, sl, addr, kind in accs:
                assert warp_of.setdefault((sl, addr), lane // 32) == lane // 32, (stage, sl, addr)
    for stage, accs in sched:
        owner = {}
        readers = defaultdict(set)
        for lane, sl, addr, kind in accs:
            assert 0 <= addr < (cpb * 18 * n if sl == "GE" else size), (stage, sl, addr, size)
            key = (sl, addr)
            if kind == "w":
                assert owner.get(key, lane) == lane, ("two writers", stage, key)
                owner[key] = lane
            else:
                readers[key].add(lane)
        for key, lane in owner.items():
            others = readers.get(key, set()) - {lane}
            assert not others, ("read/write race", stage, key, lane, sorted(others)[:4])
        # coverage: each output array of the stage is written n^3 times per cell, all distinct
        nw = sum(1 for a in accs if a[3] == "w")
        per_slot = defaultdict(int)
        for a in accs:
            if a[3] == "w":
                per_slot[a[1]] += 1
        distinct = defaultdict(set)
        for a in accs:
            if a[3] == "w":
                distinct[a[1]].add(a[2])
        for sl in per_slot:
            full = cpb * 18 * n if sl == "GE" else cpb * n ** 3
            assert per_slot[sl] == len(distinct[sl]) == full, (stage, sl, per_slot[sl])
        assert nw > 0 or stage == "I"


def test_v6_instances_cover_every_degree_dispatched():
    ns = {i[0] for i in INST}
    assert {3, 4, 5, 6, 7, 8, 9} <= ns
    assert any(i[3] for i in INST) and any(i[2] for i in INST) and any(i[4] for i in INST)
