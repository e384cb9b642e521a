"""CPU tests of the product's host layer (C++ behind the C-ABI): schedules,
chunking, cost models, tuner and the table format, against the reference's
own outputs (golden fixtures) and its unit-test properties
(proj/tests/test_core.cpp, test_schedules.cpp, test_tuner.cpp)."""
import json
import os
import random
import re
import subprocess
import tempfile

import pytest

import _oracle as O
import paper_1707_09414_b200 as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "reference_golden.json")))
HARNESS = os.path.join(ROOT, "oracle", "_ref", "ref_harness")


def as_rows(s):
    return {"prologue": s.prologue,
            "chunks": [[c.chunk_id, c.offset_bytes, c.length_bytes] for c in s.chunks],
            "events": [[r, 0 if e.kind == "send" else 1, e.peer, e.chunk, e.group]
                       for r, ops in enumerate(s.per_rank_ops) for e in ops]}


def cfg(algo, chunk=0, radix=0):
    return B.AlgorithmConfig(B.Algorithm[algo], radix, chunk)


def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "bcl.h")).read()
    declared = set(re.findall(r"\b(bcl_\w+)\s*\(", header)) - {"bcl_cost_fn"}
    out = subprocess.run(["nm", "-D", "--defined-only", B.lib_path()], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (bcl_\w+)", out))
    assert declared, "no declarations parsed"
    assert declared <= exported, declared - exported
    B.lib()  # loads without a GPU


def test_make_chunks_goldens_and_coverage():
    assert [(c.chunk_id, c.offset_bytes, c.length_bytes) for c in B.make_chunks(10, 4)] == \
        [(0, 0, 4), (1, 4, 4), (2, 8, 2)]
    assert len(B.make_chunks(1048576, 131072)) == 8
    assert [(c.offset_bytes, c.length_bytes) for c in B.make_chunks(0, 16)] == [(0, 0)]
    assert [(c.offset_bytes, c.length_bytes) for c in B.make_chunks(5, 100)] == [(0, 5)]
    with pytest.raises(ValueError):
        B.make_chunks(10, 0)
    rng = random.Random(7)  # test_core.cpp:48-67
    for _ in range(500):
        m, c = rng.randrange(1000000), 1 + rng.randrange(20000)
        ch = B.make_chunks(m, c)
        assert sum(x.length_bytes for x in ch) == m
        assert len(ch) == (1 if m == 0 else (m + c - 1) // c)
        assert [(x.chunk_id, x.offset_bytes, x.length_bytes) for x in ch] == O.make_chunks(m, c)


@pytest.mark.parametrize("idx", range(len(GOLD["schedules"])))
def test_schedules_match_reference(idx):
    g = GOLD["schedules"][idx]
    algo, n, root, m, chunk, radix = g["case"]
    got = as_rows(B.make_schedule(cfg(algo, chunk if algo == "chain_pipelined" else 0, radix), n, root, m))
    assert got == {k: g[k] for k in ("prologue", "chunks", "events")}


def test_rotation_and_validity_properties():
    rng = random.Random(3)  # test_schedules.cpp:204-253
    for _ in range(60):
        n = 1 + rng.randrange(24)
        root = rng.randrange(n)
        m = rng.randrange(10000)
        k = 2 + rng.randrange(4)
        c = 1 + rng.randrange(2048)
        for algo in ("direct", "chain", "knomial", "scatter_ring_allgather", "chain_pipelined"):
            if algo == "chain_pipelined" and n < 2:
                continue
            conf = cfg(algo, c if algo == "chain_pipelined" else 0, k if algo == "knomial" else 0)
            base = B.make_schedule(conf, n, 0, m)
            rot = B.make_schedule(conf, n, root, m)
            for l in range(n):
                a = (l + root) % n
                assert [(e.kind, (e.peer + root) % n, e.chunk, e.group) for e in base.per_rank_ops[l]] == \
                    [(e.kind, e.peer, e.chunk, e.group) for e in rot.per_rank_ops[a]]
            assert B.validate_schedule(conf, n, root, m) is None
            assert as_rows(rot) == O.schedule(algo, n, root, m, conf.chunk_bytes, conf.radix_k)


def test_schedule_contract_errors():
    with pytest.raises(ValueError):
        B.schedule_chain_pipelined(3, 0, 8, 0)
    with pytest.raises(ValueError):
        B.schedule_chain_pipelined(1, 0, 8, 4)
    with pytest.raises(ValueError):
        B.schedule_direct(3, 3, 100)
    with pytest.raises(ValueError):
        B.schedule_knomial(4, 1, 0, 100)
    assert B.to_text(cfg("knomial", radix=2), 2, 0, 100) == B.to_text(cfg("chain"), 2, 0, 100)


def test_cost_models_match_reference():
    for g in GOLD["models"]:
        assert B.cost_for(cfg("knomial", radix=2), g["n"], g["m"]) == g["costs"]["knomial"]
        assert B.cost_for(cfg("scatter_ring_allgather"), g["n"], g["m"]) == g["costs"]["scatter_ring_allgather"]
        assert B.cost_for(cfg("chain_pipelined", g["c"]), g["n"], g["m"]) == g["costs"]["chain_pipelined"]


def _pow2(lo, hi):
    v = []
    while lo <= hi:
        v.append(lo)
        lo *= 2
    return v


@pytest.mark.parametrize("idx", range(len(GOLD["tables"])))
def test_tune_tables_byte_identical_to_reference(idx):
    g = GOLD["tables"][idx]
    nl, lo, hi, cands, clo, chi, oracle = g["case"]
    if oracle != "analytical":
        pytest.skip("the simulated oracle (simengine) is out of scope; its tables are still loaded below")
    cs = [cfg(a, 0, 2 if "knomial" in a else 0) for a in cands.split(",")]
    t = B.tune([int(x) for x in nl.split(",")], _pow2(lo, hi), cs, _pow2(clo, chi))
    assert t.text() == g["csv"]


def test_select_matches_reference_on_reference_tables():
    tables = [B.load_table_text(t["csv"]) for t in GOLD["tables"]]
    for s in GOLD["selects"]:
        t = tables[s["table"]]
        for m, want in zip(s["probes"], s["answers"]):
            if want == "out_of_range":
                with pytest.raises(IndexError):
                    B.select(t, s["n"], m)
            else:
                c = B.select(t, s["n"], m)
                assert "%s %d %d" % (c.algorithm.name, c.radix_k, c.chunk_bytes) == want


def test_table_round_trip_and_parse_errors_match_reference():
    for g in GOLD["tables"]:
        t = B.load_table_text(g["csv"])
        assert t.text() == g["csv"]
        assert t.oracle == g["case"][-1]
    for p in GOLD["parse"]:
        want = p["result"][0]
        if want.startswith("parse_error"):
            with pytest.raises(B.TableParseError) as e:
                B.load_table_text(p["text"])
            assert e.value.line == int(want.split()[1])
            assert str(e.value) == want.split(" ", 2)[2]
        else:
            B.load_table_text(p["text"])


def test_measured_tables_load_in_the_reference():
    """Tables written with the Measured oracle parse in the unmodified
    reference load_table (tuner.cpp:267-345) and select identically."""
    sizes = _pow2(4, 1 << 20)
    t = B.tune_measured([2, 4], sizes, [cfg("knomial", radix=2), cfg("chain_pipelined")], _pow2(65536, 1 << 20),
                        lambda c, n, m: (2e-6 if c.algorithm == B.Algorithm.knomial else 4e-6) + m / 7e11 *
                        (2 if c.algorithm == B.Algorithm.knomial else 1) + c.chunk_bytes / 7e11,
                        provenance="unit test")
    text = t.text()
    assert text.startswith("# bcl-oracle: measured unit test\n")
    # the push-protocol rule rides in a comment line the reference skips
    lines = text.splitlines()
    lines.insert(1, "# bcl-push-from: n=4 bytes=268435456")
    lines.insert(2, "# bcl-ll128-upto: n=2 bytes=33554432")
    text = "\n".join(lines) + "\n"
    t = B.load_table_text(text)
    assert t.text() == text
    again = B.load_table_text(text)
    assert again == t and again.oracle == "measured"
    if not os.path.exists(HARNESS):
        pytest.skip("oracle/_ref not built here")
    with tempfile.NamedTemporaryFile("w", suffix=".csv", delete=False) as f:
        f.write(text)
    probes = [0, 4, 1000, 70000, 1 << 20, 1 << 30]
    out = subprocess.run([HARNESS, "select", f.name, "4", *map(str, probes)], capture_output=True,
                         text=True).stdout.splitlines()
    os.unlink(f.name)
    for m, line in zip(probes, out):
        c = B.select(t, 4, m)
        assert line == "%s %d %d" % (c.algorithm.name, c.radix_k, c.chunk_bytes)


def test_tune_contract_errors():
    cs = [cfg("knomial", radix=2), cfg("chain_pipelined")]
    with pytest.raises(ValueError):
        B.tune([], [1024], cs, [8192])
    with pytest.raises(ValueError):
        B.tune([4], [2048, 1024], cs, [8192])
    with pytest.raises(ValueError):
        B.tune([4], [1024], [cfg("chain_pipelined")], [])
    with pytest.raises(IndexError):
        B.select(B.tune([4, 8], [1024], cs, [8192]), 3, 4096)


def test_builtin_table_is_valid_and_covers_2_4_8():
    t = B.builtin_table()
    ns = sorted({e.n for e in t.entries})
    assert ns[:1] == [2]
    for n in (2, 4, 8):
        for m in (4, 4096, 1 << 20, 64 << 20, 1 << 30):
            B.select(t, n, m)


def test_builtin_table_is_the_merge_of_the_measured_tables():
    """paper_1707_09414_b200/tables/b200_default.csv (compiled into the
    library) is exactly tools/merge_tables.py over the per-n measured tables,
    and the library's builtin table carries its transport rules."""
    tdir = os.path.join(ROOT, "paper_1707_09414_b200", "tables")
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "merged.csv")
        subprocess.run(["python", os.path.join(ROOT, "tools", "merge_tables.py"), out,
                        os.path.join(tdir, "b200_measured_n2.csv"), os.path.join(tdir, "b200_measured_n4.csv"),
                        os.path.join(tdir, "b200_predicted_n8.csv")],
                       check=True, capture_output=True)
        assert open(out).read() == open(os.path.join(tdir, "b200_default.csv")).read()
    text = B.builtin_table().text()
    assert text == open(os.path.join(tdir, "b200_default.csv")).read()
    assert "# bcl-ll128-upto: n=4" in text and "# bcl-push-from: n=4" in text
    # n = 8 rows exist (so select no longer falls back to the n = 4 rows) and
    # are labelled as predicted, not measured (tools/predict_n8.py)
    assert {e.n for e in B.builtin_table().entries} == {2, 4, 8}
    assert "PREDICTED n=8" in text.splitlines()[0]


def test_call_overhead_extends_the_reference_model():
    """B200 per-call constant a0 (NetworkParams.call_overhead_s): every
    algorithm's cost gains exactly a0; a0 = 0 is the reference model; a
    uniform constant never changes the tuner's winners, only its predicted
    costs."""
    cands = [B.AlgorithmConfig.of("knomial", 2), B.AlgorithmConfig.of("scatter_ring_allgather"),
             B.AlgorithmConfig.of("chain_pipelined"), B.AlgorithmConfig.of("direct"), B.AlgorithmConfig.of("chain")]
    a0 = 17.2e-6
    for c in cands:
        cc = B.AlgorithmConfig(c.algorithm, c.radix_k, 65536 if c.algorithm == B.Algorithm.chain_pipelined else 0)
        for n in (2, 4, 8):
            for m in (0, 1, 1000, 1 << 20, 64 << 20):
                base = B.cost_for(cc, n, m, 3e-6, 7.5e11)
                assert B.cost_for(cc, n, m, 3e-6, 7.5e11, call_overhead_s=a0) == pytest.approx(base + a0, rel=1e-12)
    sizes = [4 << i for i in range(29)]
    chunks = [65536 << i for i in range(7)]
    plain = B.tune([2, 4, 8], sizes, cands[:4], chunks, startup_s=3e-6, link_Bps=7.5e11)
    withc = B.tune([2, 4, 8], sizes, cands[:4], chunks, startup_s=3e-6, link_Bps=7.5e11, call_overhead_s=a0)
    assert [(e.n, e.msg_min_bytes, e.msg_max_bytes, e.config) for e in plain.entries] == \
           [(e.n, e.msg_min_bytes, e.msg_max_bytes, e.config) for e in withc.entries]
    for a, b in zip(plain.entries, withc.entries):
        assert b.predicted_cost_s == pytest.approx(a.predicted_cost_s + a0, rel=1e-9)
    with pytest.raises(ValueError):
        B.cost_for(cands[0], 4, 100, call_overhead_s=-1.0)


def test_group_calls_without_a_gpu():
    """bcl_group_start/end are host bookkeeping: nesting works, an end without
    a start is a contract error, an empty group flushes nothing."""
    from paper_1707_09414_b200 import _lib
    lib = B.lib()
    assert lib.bcl_group_start() == 0
    assert lib.bcl_group_start() == 0
    assert lib.bcl_group_end() == 0
    assert lib.bcl_group_end() == 0
    with pytest.raises(ValueError, match="group_end without group_start"):
        _lib._check(lib.bcl_group_end())
    with B.group():
        pass


def test_config_struct_is_cached_and_value_semantics_hold():
    """AlgorithmConfig builds its C struct once (the per-call binding passes
    it by reference); equality, hashing, pickling and the struct's fields
    still follow the three dataclass fields."""
    import pickle
    a = B.AlgorithmConfig(B.Algorithm.chain_pipelined, 0, 65536)
    s1 = a._c()
    assert a._c() is s1 and (s1.algorithm, s1.radix_k, s1.chunk_bytes) == (4, 0, 65536)
    b = B.AlgorithmConfig.of("chain_pipelined", chunk_bytes=65536)
    assert a == b and hash(a) == hash(b) and {a: 1}[b] == 1
    c = pickle.loads(pickle.dumps(a))
    assert c == a and c._c().chunk_bytes == 65536
    assert B.AlgorithmConfig(B.Algorithm.knomial, 2, 0) != a
    assert repr(a) == "AlgorithmConfig(algorithm=<Algorithm.chain_pipelined: 4>, radix_k=0, chunk_bytes=65536)"
