"""CPU restatement of the reference planner/replay SUB-OPERATIONS for small
cases -- TEST INFRASTRUCTURE ONLY (the parity checker of tests/; never
imported by the product package, which runs these on the device / in the
native allocator).

Each function restates one reference function on plain tuples, citing the
file:line it follows (paths under /root/reference/pkg/src/memplan/). Pinned
against the reference's own known-answer tests (tests/test_subops_*.py carry
the same numbers) and, where the reference is importable, against it directly
(tests/test_reference_live.py).

Rectangles are tuples (id, size, t_s, t_e, addr).
"""

from __future__ import annotations


def group_keys(events):
    """planner.py:74-85: {(p_s, p_e): members sorted by (t_s, id)}, keys in
    PhaseId order. events: (id, t_s, p_s, p_e) with comparable phase keys."""
    out = {}
    for e in events:
        out.setdefault((e[2], e[3]), []).append(e)
    return [(k, sorted(out[k], key=lambda e: (e[1], e[0]))) for k in sorted(out)]


def tmp_of(rects, height, t_lo, t_hi):
    """planner.py:110-115: Python int / int of the used area over the box."""
    used = sum(r[1] * (r[3] - r[2]) for r in rects)
    return used / (height * (t_hi - t_lo))


def plan_box(rects):
    """planner.py:88-95: (height, t_lo, t_hi, tmp) of placed rectangles."""
    h = max(r[4] + r[1] for r in rects)
    lo = min(r[2] for r in rects)
    hi = max(r[3] for r in rects)
    return h, lo, hi, tmp_of(rects, h, lo, hi)


def weighted(tmps_weights):
    """planner.py:118-121 with CPython semantics: float * int products,
    builtin sum, / int."""
    return sum(t * w for t, w in tmps_weights) / sum(w for _, w in tmps_weights)


def fuse(larger, smaller):
    """planner.py:124-169: addresses of `smaller`'s rectangles placed into
    `larger` by the cursor walk; returns {id: addr} and the placement order."""
    fixed = list(larger)
    anchors = sorted({r[4] for r in larger})
    todo = sorted(smaller, key=lambda r: (r[2], r[0]))
    cur = anchors[0]
    placed, order = {}, []

    def clash(r, a):
        return any(f[4] < a + r[1] and a < f[4] + f[1] and f[2] < r[3] and r[2] < f[3] for f in fixed)

    while todo:
        k = next((i for i, r in enumerate(todo) if not clash(r, cur)), None)
        if k is None:
            higher = [a for a in anchors if a > cur]
            cur = higher[0] if higher else max(f[4] + f[1] for f in fixed)
            continue
        r = todo.pop(k)
        placed[r[0]] = cur
        order.append(r[0])
        fixed.append((r[0], r[1], r[2], r[3], cur))
        cur += r[1]
    return placed, order


def alg1(items):
    """planner.py:236-254: items (t_s, t_e, tie) -> layer index per item, in
    input order; layer count."""
    ends = []
    out = [None] * len(items)
    for k in sorted(range(len(items)), key=lambda k: (items[k][0], items[k][2])):
        s, e, _ = items[k]
        best = None
        for li, end in enumerate(ends):
            if end < s and (best is None or end > ends[best]):
                best = li
        if best is None:
            ends.append(e)
            best = len(ends) - 1
        else:
            ends[best] = max(ends[best], e)
        out[k] = best
    return out, len(ends)


def closed_overlap(spans):
    """Max number of closed intervals sharing a point (the layer-count optimum)."""
    return max(sum(1 for s, e in spans if s <= p <= e) for p, _ in spans)


class Cache:
    """baseline.py:35-95: best fit over all blocks in (segment, address)
    order, split, merge; power-of-two segments >= min_segment."""

    def __init__(self, base=0, min_segment=2 * 1024 * 1024):
        self.next_base = base
        self.min_segment = min_segment
        self.segs = []  # [base, size, [(lo, hi), ...]]
        self.live = {}
        self.reserved = 0

    def malloc(self, rid, size):
        best = None
        for g, seg in enumerate(self.segs):
            for i, (lo, hi) in enumerate(seg[2]):
                if hi - lo >= size and (best is None or hi - lo < best[2]):
                    best = (g, i, hi - lo)
        grown = 0
        if best is None:
            ss = max(self.min_segment, 1 << (size - 1).bit_length())
            self.segs.append([self.next_base, ss, [(self.next_base, self.next_base + ss)]])
            self.next_base += ss
            self.reserved += ss
            grown = ss
            best = (len(self.segs) - 1, 0, ss)
        g, i, _ = best
        lo, hi = self.segs[g][2].pop(i)
        if lo + size < hi:
            self.segs[g][2].insert(i, (lo + size, hi))
        self.live[rid] = (g, lo, size)
        return lo, grown

    def free(self, rid):
        g, lo, size = self.live.pop(rid)
        blocks = self.segs[g][2]
        blocks.append((lo, lo + size))
        blocks.sort()
        merged = []
        for b in blocks:
            if merged and merged[-1][1] == b[0]:
                merged[-1] = (merged[-1][0], b[1])
            else:
                merged.append(b)
        self.segs[g][2] = merged
        return lo, size


def reuse_best_fit(free, space, size):
    """sim.py:120-140: lowest address of the smallest piece of free ∩ space
    holding size (ties: lowest address), or None."""
    pieces = []
    for a, b in free:
        for c, d in space:
            lo, hi = max(a, c), min(b, d)
            if hi > lo:
                pieces.append((hi - lo, lo))
    fits = sorted(p for p in pieces if p[0] >= size)
    return fits[0][1] if fits else None


def metrics(log):
    """sim.py:67-117 over a list of log dicts: the SimReport fields as a dict."""
    pool = live = cache = peak = cpeak = reserved = fb = mm = ru = 0
    for r in log:
        k = r["kind"]
        if k == "init":
            pool = r["pool_size"]
        elif k == "reserve":
            reserved += r["bytes"]
        elif k == "alloc":
            live += r["size"]
            peak = max(peak, live)
            if r["space"] == "cache":
                cache += r["size"]
                cpeak = max(cpeak, cache)
            fb += r["route"] in ("fallback", "mismatch")
            mm += r["route"] == "mismatch"
            ru += r["route"] == "reuse"
        elif k == "free":
            live -= r["size"]
            if r["space"] == "cache":
                cache -= r["size"]
    rp = pool + reserved
    eff = peak / rp if rp else 1.0
    return dict(allocated_peak=peak, reserved_peak=rp, efficiency=eff, fragmentation=1.0 - eff, pool_size=pool,
                fallback_count=fb, fallback_bytes_peak=cpeak, reuse_hits=ru, mismatch_count=mm)
