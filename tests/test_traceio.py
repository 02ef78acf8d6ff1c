"""Trace and plan files through the native reader/writer (libstw_io.so).

Known answers restate the reference's pins (pkg/tests/test_traceio.py:26-173);
byte identity of written files is pinned by sha256 fixtures the reference
produced (tests/golden/make_traceio_golden.py -> traceio.json) and, where the
reference is importable, checked live together with an error-path fuzz that
compares exception type and message with the reference's on corrupted files."""

import hashlib
import json
import os
import random

import pytest

import paper_2507_16274_b200 as M
from paper_2507_16274_b200 import tracegen
from paper_2507_16274_b200.traceio import parse_trace, read_plan, write_plan, write_trace

from conftest import GOLDEN, HAVE_REF, ref

HEADER = '{"kind":"trace","version":1,"format":"raw"}'
A1 = '{"op":"alloc","id":1,"size":1024,"phase":"F:0","module":"","dynamic":false}'


def put(path, *lines):
    path.write_text("\n".join(lines) + "\n", encoding="utf-8")
    return path


def test_pairing_and_persistent(tmp_path):
    tr = parse_trace(put(tmp_path / "t.jsonl", HEADER, A1, '{"op":"free","id":1,"phase":"B:0","module":""}'))
    (ev,) = tr.events
    assert (ev.size, ev.t_s, ev.t_e, ev.p_s.tag(), ev.p_e.tag(), ev.dynamic) == (1024, 0, 1, "F:0", "B:0", False)
    tr = parse_trace(put(tmp_path / "u.jsonl", HEADER, A1,
                         '{"op":"alloc","id":2,"size":512,"phase":"B:0","module":"","dynamic":false}',
                         '{"op":"free","id":2,"phase":"B:0","module":""}'))
    ev = next(e for e in tr.events if e.id == 1)
    assert ev.t_e == tr.horizon == 3 and ev.p_e.tag() == "B:0"


@pytest.mark.parametrize("lines,match", [
    ([HEADER, A1.replace("false", "true")], "dynamic event missing layer"),
    ([HEADER, "{not json"], ":2:"),
    ([HEADER, '{"op":"free","id":9,"phase":"F:0","module":""}'], "free without matching alloc"),
    ([HEADER, A1, A1], "duplicate alloc id"),
    (['{"kind":"trace","version":99,"format":"raw"}'], "version"),
])
def test_rejections(tmp_path, lines, match):
    with pytest.raises(M.TraceError, match=match):
        parse_trace(put(tmp_path / "t.jsonl", *lines))


def test_sizes_rounded_up(tmp_path):
    tr = parse_trace(put(tmp_path / "t.jsonl", HEADER, A1.replace("1024", "100"),
                         '{"op":"free","id":1,"phase":"F:0","module":""}'))
    assert tr.events[0].size == 512


@pytest.mark.parametrize("preset", ["dense", "dense_vpp", "moe", "moe_recompute"])
@pytest.mark.parametrize("form", ["raw", "paired"])
def test_round_trip_and_golden_bytes(tmp_path, preset, form):
    trace = M.synth_trace(tracegen.SynthConfig.for_preset(preset, seed=11))
    p1, p2 = tmp_path / "a.jsonl", tmp_path / "b.jsonl"
    write_trace(trace, p1, form=form)
    again = parse_trace(p1)
    write_trace(again, p2, form=form)
    assert p1.read_bytes() == p2.read_bytes()
    assert again.events == trace.events
    assert again.phase_schedule == trace.phase_schedule and again.layer_schedule == trace.layer_schedule
    with open(os.path.join(GOLDEN, "traceio.json")) as fh:
        want = json.load(fh)["trace"][f"{preset}/11/{form}"]
    assert hashlib.sha256(p1.read_bytes()).hexdigest() == want


def _bundle(pool=4096):
    return M.PlanBundle(4096 if pool is None else pool, 512,
                        (M.PlanDecision(0, 0, 1024, 0, 3), M.PlanDecision(1, 1024, 512, 1, 2)),
                        {("a", "b"): M.IntervalSet([M.Interval(1536, 4096)])})


def test_plan_files(tmp_path):
    p = tmp_path / "plan.json"
    write_plan(_bundle(), p)
    got = read_plan(p)
    assert (got.pool_size, got.alignment, got.decisions, got.reuse) == (4096, 512, _bundle().decisions, _bundle().reuse)
    write_plan(got, tmp_path / "p2.json")
    assert p.read_bytes() == (tmp_path / "p2.json").read_bytes()
    write_plan(M.PlanBundle(0, 512, (), {}), tmp_path / "e.json")
    e = read_plan(tmp_path / "e.json")
    assert e.pool_size == 0 and e.decisions == () and json.loads((tmp_path / "e.json").read_text())["decisions"] == []
    doc = json.loads(p.read_text())
    doc["decisions"][0]["addr"] = 4096
    p.write_text(json.dumps(doc))
    with pytest.raises(M.PlanError, match="out of pool"):
        read_plan(p)
    doc["decisions"][0]["addr"] = 0
    doc["version"] = 2
    p.write_text(json.dumps(doc))
    with pytest.raises(M.PlanError, match="version"):
        read_plan(p)


def test_plan_golden_bytes(tmp_path):
    trace = M.synth_trace(tracegen.SynthConfig.for_preset("moe_recompute", seed=1))
    with open(os.path.join(GOLDEN, "traceio.json")) as fh:
        want = json.load(fh)["plan_fixture"]
    # the bundle is rebuilt from the fixture (no device needed): decisions + reuse as the reference wrote them
    b = M.PlanBundle(want["pool_size"], 512, tuple(M.PlanDecision(*d) for d in want["decisions"]),
                     {tuple(k): M.IntervalSet([M.Interval(a, c) for a, c in v]) for k, v in want["reuse"]})
    write_plan(b, tmp_path / "p.json")
    assert hashlib.sha256((tmp_path / "p.json").read_bytes()).hexdigest() == want["sha256"]
    assert len(trace.events) > 0


# ---------------------------------------------------------------------------
# live comparison with the reference (build container only)


def _outcome(fn, path):
    try:
        r = fn(path)
    except Exception as exc:  # noqa: BLE001 -- the comparison is the point
        return ("raise", type(exc).__name__, str(exc))
    if hasattr(r, "phase_schedule"):
        return ("ok", [(e.id, e.size, e.t_s, e.t_e, e.p_s.tag(), e.p_e.tag(), e.dynamic, e.l_s, e.l_e)
                       for e in r.events],
                [(s.phase.tag(), s.start, s.end) for s in r.phase_schedule],
                [(s.name, s.start, s.end) for s in r.layer_schedule])
    return ("ok", r.pool_size, r.alignment, [tuple(vars(d).values()) if hasattr(d, "__dict__") else
                                             (d.id, d.addr, d.size, d.t_s, d.t_e) for d in r.decisions],
            sorted((k, [(iv.lo, iv.hi) for iv in v]) for k, v in r.reuse.items()))


_VALUES = ['0', '-1', '1.5', '"7"', '" 12 "', '"1_0"', '"x"', 'null', 'true', '[]', '{}', '"F:1"', '"B:0.2"',
           '"init"', '"opt"', '"F:x"', '1e3', '"\\u00e9"', '""', '"F:0"', '3']


def _mutate(rng, lines):
    lines = list(lines)
    k = rng.randrange(len(lines))
    r = rng.random()
    if r < 0.15 and len(lines) > 1:
        del lines[k]
    elif r < 0.25:
        lines.insert(k, lines[rng.randrange(len(lines))])
    elif r < 0.3:
        lines[k] = lines[k][: rng.randrange(len(lines[k]) + 1)]
    elif r < 0.35 and len(lines) > 2:
        j = rng.randrange(len(lines))
        lines[k], lines[j] = lines[j], lines[k]
    else:
        try:
            obj = json.loads(lines[k])
        except ValueError:
            return lines
        if isinstance(obj, dict) and obj:
            key = rng.choice(sorted(obj))
            if rng.random() < 0.2:
                del obj[key]
                lines[k] = json.dumps(obj)
            else:
                text = json.dumps(obj)
                val = rng.choice(_VALUES)
                head = json.dumps({key: obj[key]})[1:-1]
                lines[k] = text.replace(head, head.split(":", 1)[0] + ":" + val, 1)
    return lines


@pytest.mark.skipif(not HAVE_REF, reason="reference not present")
@pytest.mark.parametrize("form", ["raw", "paired"])
def test_error_fuzz_matches_reference(tmp_path, form):
    R = ref()
    rng = random.Random(17 if form == "raw" else 18)
    base = tmp_path / "base.jsonl"
    R.write_trace(R.synth_trace(R.SynthConfig.for_preset("moe_recompute", seed=3, num_layers=2,
                                                         num_microbatches=1)), base, form=form)
    lines = base.read_text().splitlines()
    for i in range(300):
        mutated = lines
        for _ in range(rng.randint(1, 3)):
            mutated = _mutate(rng, mutated)
        p = tmp_path / f"m{i}.jsonl"
        p.write_text("\n".join(mutated) + "\n")
        assert _outcome(parse_trace, p) == _outcome(R.parse_trace, p), (i, p.read_text()[:2000])


@pytest.mark.skipif(not HAVE_REF, reason="reference not present")
def test_plan_fuzz_matches_reference(tmp_path):
    R = ref()
    rng = random.Random(5)
    tr = R.synth_trace(R.SynthConfig.for_preset("moe", seed=2, num_layers=2, num_microbatches=1))
    plan, rmap = R.plan_trace(tr)
    base = tmp_path / "plan.json"
    R.write_plan(plan.to_bundle(rmap), base)
    mine = tmp_path / "mine.json"
    write_plan(read_plan(base), mine)
    assert mine.read_bytes() == base.read_bytes()
    doc = json.loads(base.read_text())
    for i in range(200):
        d = json.loads(json.dumps(doc))
        for _ in range(rng.randint(1, 2)):
            where = rng.random()
            val = json.loads(rng.choice(_VALUES[:-3]))
            if where < 0.4 and d["decisions"]:
                dec = rng.choice(d["decisions"])
                dec[rng.choice(sorted(dec))] = val
            elif where < 0.6 and d["reuse_map"]:
                e = rng.choice(d["reuse_map"])
                if e["intervals"] and rng.random() < 0.5:
                    e["intervals"][0][rng.randrange(2)] = val
                else:
                    e[rng.choice(["l_s", "l_e"])] = val
            else:
                d[rng.choice(["version", "pool_size", "alignment"])] = val
        p = tmp_path / f"p{i}.json"
        p.write_text(json.dumps(d, indent=rng.choice([None, 2])))
        assert _outcome(read_plan, p) == _outcome(R.read_plan, p), (i, p.read_text()[:500])
