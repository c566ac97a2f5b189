"""LL128 protocol geometry, host side (no GPU): the library's own inbox layout
and planner (lane_ll128.cuh layout128 / plan128 through the C ABI's
host-only queries).

* Every (inbox, slot, chunk, sub-part, line) of a call maps to its own line
  and the lines tile the parity set exactly — no two packets of one call
  share a line (a shared line would let one overwrite the other's epoch
  word) and nothing falls outside the set the call was sized for.
* Within LL128's range, every layout / k / size / CTA budget the library
  plans fits the per-set capacity allocated at init, so the protocol never
  silently falls back, and the plan covers the message.
"""
import ctypes
import itertools

import pytest

from paper_2508_13397_b200 import _lib

LAYOUTS = [(1, 2), (2, 1), (2, 2), (1, 4), (4, 1), (2, 4), (4, 2), (8, 1), (1, 8), (3, 2), (2, 3)]
M_BYTES, CG_MIN_BYTES = 32 << 20, 16 << 10  # LANE_LL128_MAX_BYTES, LANE_LL128_MIN_CHUNK_BYTES defaults


def line(N, G, cap, lu, kind, slot, c, b, ln):
    out = ctypes.c_int64()
    code = _lib.load().lane_ll128_line_query(N, G, cap, lu, kind, slot, c, b, ln, ctypes.byref(out))
    return code, out.value


def plan(N, G, k, ng, C, m=M_BYTES, cgm=CG_MIN_BYTES):
    out = (ctypes.c_int64 * 6)()
    assert _lib.load().lane_ll128_plan_query(N, G, k, ng, C, m, cgm, out) == 0
    return dict(zip(("C", "cg", "cap", "lu", "need", "set"), list(out)))


@pytest.mark.parametrize("N,G", LAYOUTS)
def test_layout_tiles_the_set_exactly(N, G):
    for cap, lu in itertools.product((1, 3), (1, 2, 5)):
        seen = []
        for kind in (1, 2, 3, 4):
            slots = G - 1 if kind in (1, 4) else N
            subparts = N if kind in (1, 4) else 1
            for s, c, b, ln in itertools.product(range(slots), range(cap), range(subparts), range(lu)):
                code, idx = line(N, G, cap, lu, kind, s, c, b, ln)
                assert code == 0
                seen.append(idx)
        assert sorted(seen) == list(range(2 * G * N * cap * lu)), (N, G, cap, lu)


@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_ring_layout_tiles_the_set_exactly(P):
    for cap, lp in itertools.product((1, 4), (1, 3)):
        seen = []
        for kind in (5, 6):
            for s, c, ln in itertools.product(range(P - 1), range(cap), range(lp)):
                code, idx = line(1, P, cap, lp, kind, s, c, 0, ln)
                assert code == 0
                seen.append(idx)
        assert sorted(seen) == list(range(2 * (P - 1) * cap * lp)), (P, cap, lp)


def test_line_query_rejects_out_of_range():
    assert line(2, 2, 1, 1, 1, 1, 0, 0, 0)[0] == -1  # G-1 = 1 L1 slot
    assert line(2, 2, 1, 1, 2, 2, 0, 0, 0)[0] == -1  # N = 2 L2 slots
    assert line(2, 2, 2, 3, 3, 0, 2, 0, 0)[0] == -1  # chunk
    assert line(2, 2, 2, 3, 4, 0, 0, 2, 0)[0] == -1  # sub-part
    assert line(2, 2, 2, 3, 4, 0, 0, 0, 3)[0] == -1  # line
    assert line(2, 2, 2, 3, 7, 0, 0, 0, 0)[0] == -1  # kind
    assert line(2, 2, 2, 3, 5, 3, 0, 0, 0)[0] == -1  # ring slot (P - 1 = 3 slots)


def _sizes():
    out = set()
    for e in range(16, 22):  # 1 MiB .. 32 MiB of message, in granules, plus ragged neighbours
        g = 1 << e
        out |= {g, g + 3, 3 * g // 2 + 1, g - 5}
    return sorted(s for s in out if (1 << 16) <= s <= M_BYTES // 16)


@pytest.mark.parametrize("N,G", [(2, 1), (1, 2), (2, 2), (4, 1), (1, 4), (2, 4), (4, 2), (8, 1), (1, 8)])
def test_plans_fit_and_cover_in_the_ll128_range(N, G):
    P = N * G
    for k in (1, 2, 4, 8, 16):
        for C0 in sorted({max(148 // k, 1), max(148 // (P * k), 1), 1}):  # multi-GPU, emulated, 1 CTA
            for ng in _sizes():
                p = plan(N, G, k, ng, C0)
                ctx = (N, G, k, C0, ng, p)
                assert p["need"] <= p["set"], ctx  # LL128 never falls back inside its range
                assert 1 <= p["C"] <= C0, ctx
                assert p["cg"] >= CG_MIN_BYTES // 16 or p["cg"] >= -(-ng // k), ctx
                slice0 = -(-ng // k)
                assert p["cap"] >= k * 1 and p["cap"] * p["cg"] >= ng, ctx  # the chunks cover the message
                assert p["cap"] >= k * (-(-slice0 // p["cg"])) - k, ctx
                su = -(-(-(-p["cg"] // G)) // N)
                # line pairs of 15 granules cover the largest sub-part, no spare pair
                assert p["lu"] % 2 == 0 and p["lu"] // 2 * 15 >= su > (p["lu"] // 2 - 1) * 15, ctx
