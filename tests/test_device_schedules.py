"""CPU checks of the evaluation orders the CUDA kernels use in place of the
oracle's loops.  The device code is bit-exact
only if these schedules perform exactly the oracle's operations on exactly the
oracle's operands; here each schedule is replayed symbolically and compared
with the oracle's expression tree.

* lane_canon32 (csrc/device.cuh): a width-32 canonical sum evaluated by one
  lane -- leaves in 5-bit bit-reversed order, a merge stack, empty right
  subtrees skipped -- against canon_sum of oracle/orc_tracker.hpp.
* warp_canon (csrc/mgs_warp.cuh): the warp-resident MGS sum for
  width_mgs(N) in {32, 64} (lane-local level, five shuffle levels) against
  canon_sum.
* mono_pair (csrc/device.cuh): the two-lane reverse-mode schedule of a long
  monomial against Table 1: same products, same operand
  order, no slot read before it is written by the partner.
"""
import pytest


def canon_sum(K, P):
    """oracle canon_sum as an expression tree (nested tuples ('+', l, r))."""
    part = []
    for p in range(min(P, K)):
        acc = f"c{p}"
        r = p + P
        while r < K:
            acc = ("+", acc, f"c{r}")
            r += P
        part.append(acc)
    off = P // 2
    while off >= 1:
        for p in range(off):
            if p + off < K:
                part[p] = ("+", part[p], part[p + off])
        off //= 2
    return part[0]


def brev5(t):
    return int(f"{t:05b}"[::-1], 2)


def popc(t):
    return bin(t).count("1")


def ctz(x):
    n = 0
    while x % 2 == 0 and n < 5:
        x //= 2
        n += 1
    return n


def lane_canon32(K):
    """Replay of lane_canon32: stack positions depend on t only."""
    st, ne = [None] * 6, [False] * 6
    for t in range(32):
        p = brev5(t)
        d = popc(t)
        v = None
        if p < K:
            v = f"c{p}"
            r = p + 32
            while r < K:
                v = ("+", v, f"c{r}")
                r += 32
        st[d], ne[d] = v, p < K
        for m in range(ctz(t + 1)):
            top = d - m
            if ne[top]:
                st[top - 1] = ("+", st[top - 1], st[top])
    return st[0]


@pytest.mark.parametrize("K", list(range(1, 70)) + [96, 127, 128, 200, 511, 512])
def test_lane_canon32_is_the_canonical_tree(K):
    assert lane_canon32(K) == canon_sum(K, 32)


def warp_canon(N):
    """Replay of warp_canon for E = ceil(N/32) <= 4 (lane l holds rows l + 32 r)."""
    E = (N + 31) // 32
    P = 32 if E <= 2 else 64
    acc = {}
    for lane in range(32):
        rows = [lane + 32 * r for r in range(E)]
        v = [f"c{i}" if i < N else None for i in rows]
        a = v[0]
        if P == 32:
            for r in range(1, E):
                if lane + 32 * r < N:
                    a = ("+", a, v[r])
        else:
            if E > 2 and lane + 64 < N:
                a = ("+", a, v[2])
            if E > 1:
                a1 = v[1]
                if E > 3 and lane + 96 < N:
                    a1 = ("+", a1, v[3])
                a = ("+", a, a1)
        acc[lane] = a
    for off in (16, 8, 4, 2, 1):
        nxt = dict(acc)
        for lane in range(32):
            if lane < off and lane + off < N:
                nxt[lane] = ("+", acc[lane], acc[lane + off])
        acc = nxt
    return acc[0]


def width_mgs(N):
    p = 1
    while p < (N + 1) // 2:
        p *= 2
    return min(256, max(32, p))


@pytest.mark.parametrize("N", list(range(1, 129)))
def test_warp_canon_is_the_canonical_tree(N):
    assert warp_canon(N) == canon_sum(N, width_mgs(N))


def mono_reference(m):
    """Table 1 products for m >= 3 as {slot: (op, a, b)} (F/B as symbols)."""
    ops = {}
    F = ["y0"]
    for k in range(1, m - 1):
        F.append(("*", F[-1], f"y{k}"))
    ops[0] = ("*", F[m - 2], f"y{m-1}")
    ops[m] = F[m - 2]
    B = f"y{m-1}"
    for k in range(m - 2, 0, -1):
        ops[k + 1] = ("*", F[k - 1], B)
        B = ("*", f"y{k}", B)
    ops[1] = B
    return ops


def mono_pair(m):
    """Replay of mono_pair: two lanes, per step phase 1 (chain + park), barrier,
    phase 2 (partials from the middle on).  Checks read-after-write order."""
    slots, written_at = {}, {}
    c = {True: "y0", False: f"y{m-1}"}
    for s in range(0, m - 1):
        for fwd in (True, False):
            if s > 0:
                c[fwd] = ("*", c[fwd], f"y{s}") if fwd else ("*", f"y{m-1-s}", c[fwd])
        phase2 = []
        for fwd in (True, False):
            k = s + 1 if fwd else m - 2 - s
            a, b = k - 1, m - 2 - k
            edge = k == m - 1 if fwd else k == 0
            mine_later = a > b if fwd else a <= b
            slot = (m if edge else k + 1) if fwd else (1 if edge else k + 1)
            if edge or not mine_later:
                slots[slot] = c[fwd]
                written_at[slot] = (s, 1)
            if 2 * s >= m - 3 and not edge and mine_later:
                phase2.append((fwd, k))
        for fwd, k in phase2:
            # the partner parked the other operand in this or an earlier step, before the barrier
            assert written_at.get(k + 1, (10 ** 9, 0)) <= (s, 1), (m, s, k)
            o = slots[k + 1]
            slots[k + 1] = ("*", c[fwd], o) if fwd else ("*", o, c[fwd])
    slots[0] = ("*", c[True], f"y{m-1}")
    return slots


@pytest.mark.parametrize("m", list(range(3, 40)) + [64, 255, 256])
def test_mono_pair_matches_table1(m):
    assert mono_pair(m) == mono_reference(m)
