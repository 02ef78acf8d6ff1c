"""Shared helpers for the parity tests (digests identical to tests/golden/make_golden.py)."""

import gzip
import hashlib
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
ROUTES = ("planned", "reuse", "fallback", "mismatch", "online")
KIND = {0: "init", 1: "reserve", 2: "alloc", 3: "free"}


def anchors():
    with open(os.path.join(GOLDEN, "anchors.json")) as fh:
        return json.load(fh)


def fuzz_fixtures():
    with gzip.open(os.path.join(GOLDEN, "fuzz.json.gz"), "rt") as fh:
        return json.load(fh)


def trace_digest(ta) -> str:
    h = hashlib.sha256()
    ph, names = ta.phases, ta.layer_names
    for i in range(len(ta)):
        d = bool(ta.dyn[i])
        ls = names[ta.ls[i]] if d else None
        le = names[ta.le[i]] if d else None
        h.update(f"{ta.id[i]},{ta.size[i]},{ta.t_s[i]},{ta.t_e[i]},{ph[ta.ps[i]].tag()},{ph[ta.pe[i]].tag()},"
                 f"{int(d)},{ls},{le};".encode())
    for s in ta.phase_spans():
        h.update(f"{s.phase.tag()},{s.start},{s.end};".encode())
    for s in ta.layer_spans():
        h.update(f"{s.name},{s.start},{s.end};".encode())
    return h.hexdigest()[:16]


def log_digest(log) -> str:
    return hashlib.sha256("\n".join(json.dumps(r, sort_keys=True, separators=(",", ":")) for r in log).encode()).hexdigest()[:16]


def oracle_log_dicts(lg, ta):
    evkey = {int(ta.id[i]): [ta.layer_names[ta.ls[i]], ta.layer_names[ta.le[i]]] for i in np.nonzero(ta.dyn)[0]}
    out = []
    for k in range(len(lg["kind"])):
        kind = KIND[int(lg["kind"][k])]
        if kind == "init":
            out.append({"kind": "init", "pool_size": int(lg["size"][k])})
        elif kind == "reserve":
            out.append({"kind": "reserve", "t": int(lg["t"][k]), "bytes": int(lg["size"][k])})
        else:
            r = {"kind": kind, "t": int(lg["t"][k]), "id": int(lg["id"][k]), "size": int(lg["size"][k]),
                 "space": "pool" if lg["space"][k] == 0 else "cache", "addr": int(lg["addr"][k])}
            if kind == "alloc":
                r["route"] = ROUTES[int(lg["route"][k])]
                if r["id"] in evkey:
                    r["key"] = evkey[r["id"]]
            out.append(r)
    return out


def plan_sha16(pool, alignment, ids, addrs, sizes, ts, te, reuse_items) -> str:
    """sha256[:16] of the reference's write_plan bytes (traceio.py:334-354)."""
    doc = {
        "version": 1, "pool_size": int(pool), "alignment": int(alignment),
        "decisions": [{"id": int(i), "addr": int(a), "size": int(s), "t_s": int(x), "t_e": int(y)}
                      for i, a, s, x, y in zip(ids, addrs, sizes, ts, te)],
        "reuse_map": [{"l_s": k[0], "l_e": k[1], "intervals": [[int(lo), int(hi)] for lo, hi in ivs]}
                      for k, ivs in sorted(reuse_items)],
    }
    return hashlib.sha256((json.dumps(doc, sort_keys=True, indent=2) + "\n").encode()).hexdigest()[:16]


def static_order(ta):
    """Static event indices in (t_s, id) order (the order of plan.decisions)."""
    idx = np.nonzero(ta.dyn == 0)[0]
    return idx[np.lexsort((ta.id[idx], ta.t_s[idx]))]


def reuse_windows(ta):
    keys, _ = ta.dynamic_keys()
    spans = {s.name: s for s in ta.layer_spans()}
    return keys, np.asarray([spans[a].start for a, _ in keys], np.int64), np.asarray([spans[b].end for _, b in keys], np.int64)


def oracle_bundle_inputs(ta, keys, off, lo, hi):
    names, kidx = ta.dynamic_keys()
    pos = {k: i for i, k in enumerate(keys)}
    key = np.array([pos.get(names[k], -1) if k >= 0 else -1 for k in kidx], np.int32)
    return key, off, lo, hi
