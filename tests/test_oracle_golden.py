"""Pins the C oracle (oracle/bcast_oracle.c) against the reference's own
outputs (tests/golden/reference_golden.json, produced by
tests/golden/make_golden.py from the unmodified reference library)."""
import json
import os

import pytest

import _oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))


def test_make_chunks_goldens():
    # proj/tests/test_core.cpp:14-46
    assert O.make_chunks(10, 4) == [(0, 0, 4), (1, 4, 4), (2, 8, 2)]
    assert O.make_chunks(8, 8) == [(0, 0, 8)]
    assert O.make_chunks(1048576, 131072) == [(i, i * 131072, 131072) for i in range(8)]
    assert O.make_chunks(5, 100) == [(0, 0, 5)]
    assert O.make_chunks(0, 16) == [(0, 0, 0)]
    with pytest.raises(ValueError):
        O.make_chunks(10, 0)


@pytest.mark.parametrize("idx", range(len(GOLD["schedules"])))
def test_schedule_matches_reference(idx):
    g = GOLD["schedules"][idx]
    algo, n, root, m, chunk, radix = g["case"]
    got = O.schedule(algo, n, root, m, chunk, radix)
    assert got["prologue"] == g["prologue"]
    assert got["chunks"] == g["chunks"]
    assert got["events"] == g["events"]


@pytest.mark.parametrize("idx", range(len(GOLD["bcasts"])))
def test_bcast_matches_reference(idx):
    g = GOLD["bcasts"][idx]
    algo, n, root, m, chunk, radix, seed = g["case"]
    payload = O.payload(seed, m)
    assert "%016x" % O.fnv(payload) == g["payload_fnv"]
    bufs = [bytearray(m) for _ in range(n)]
    bufs[root][:] = payload
    O.bcast(algo, n, root, bufs, chunk, radix)
    assert ["%016x" % O.fnv(bytes(b)) for b in bufs] == g["rank_fnv"]


def _cands(s):
    return [(a, 2 if "knomial" in a else 0) for a in s.split(",")]


def _pow2(lo, hi):
    out = []
    while lo <= hi:
        out.append(lo)
        lo *= 2
    return out


@pytest.mark.parametrize("idx", range(len(GOLD["tables"])))
def test_tune_matches_reference(idx):
    g = GOLD["tables"][idx]
    nl, lo, hi, cands, clo, chi, oracle = g["case"]
    if oracle != "analytical":
        pytest.skip("the oracle restates the analytical cost path only")
    entries = O.tune([int(x) for x in nl.split(",")], _pow2(lo, hi), _cands(cands), _pow2(clo, chi))
    assert O.save_table(entries) == g["csv"]


def test_select_matches_reference():
    for s in GOLD["selects"]:
        entries, _ = O.load_table(GOLD["tables"][s["table"]]["csv"])
        for m, want in zip(s["probes"], s["answers"]):
            got = O.select(entries, s["n"], m)
            assert (got is None and want == "out_of_range") or (got is not None and "%s %d %d" % got == want), (s["n"], m)


def test_parse_errors_match_reference():
    for p in GOLD["parse"]:
        entries, info = O.load_table(p["text"])
        want = p["result"][0]
        if want.startswith("parse_error"):
            assert entries is None, p["text"]
            assert info == int(want.split()[1]), p["text"]
        else:
            assert entries is not None, p["text"]


def test_cost_models_match_reference():
    for g in GOLD["models"]:
        assert O.cost("knomial", g["n"], g["m"], radix=2) == g["costs"]["knomial"]
        assert O.cost("scatter_ring_allgather", g["n"], g["m"]) == g["costs"]["scatter_ring_allgather"]
        assert O.cost("chain_pipelined", g["n"], g["m"], chunk=g["c"]) == g["costs"]["chain_pipelined"]
    # Eq. 5 golden, proj/tests/test_models.cpp:62-63
    assert abs(O.cost("chain_pipelined", 4, 1000000, chunk=125000) - 1.26e-3) < 1e-15
