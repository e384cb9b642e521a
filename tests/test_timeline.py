"""CPU tests of the device-timeline export (paper_1707_09414_b200/timeline.py):
per-lane %globaltimer records folded into the reference simulator's trace CSV
schema (proj/src/simengine.cpp:295-305), checked on synthetic records and
against the header the unmodified reference writes (oracle/_ref)."""
import os
import subprocess
import tempfile

import numpy as np
import pytest

from paper_1707_09414_b200.timeline import chain_rows, trace_words, write_csv

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HARNESS = os.path.join(ROOT, "oracle", "_ref", "ref_harness")


def synthetic(lanes, per_lane, plan, t0=1_000_000):
    """Lane l pulls slice l % Q of chunks c = l // Q + k * (lanes // Q)."""
    rec = np.zeros((lanes, per_lane, 4), dtype=np.int64)
    q, k_chunks = plan["slices"], plan["n_chunks"]
    ns = lanes // q
    for lane in range(lanes):
        rec[lane, per_lane - 1, 0] = t0 + lane  # enter
        for k in range(per_lane - 1):
            c = lane // q + k * ns
            if c >= k_chunks:
                break
            base = t0 + 1000 * (c + 1) + 10 * (lane % q)
            rec[lane, k] = (base, base + 400, base + 500, base + 600)
    return rec.reshape(-1)


def test_chain_rows_fold_slices_into_chunk_events():
    lanes, per_lane = 8, 6
    plan = {"slices": 2, "slice_bytes": 64, "n_chunks": 10, "ctas": 1}
    rec = synthetic(lanes, per_lane, plan)
    assert rec.size == trace_words(lanes, per_lane)
    head = chain_rows(rec, lanes, per_lane, plan, n=3, root=0, rank=0)
    assert [r[2] for r in head] == ["send"] * 10 and [r[4] for r in head] == list(range(10))
    mid = chain_rows(rec, lanes, per_lane, plan, n=3, root=0, rank=1)
    recv = [r for r in mid if r[2] == "recv"]
    send = [r for r in mid if r[2] == "send"]
    assert [r[4] for r in recv] == list(range(10)) and len(send) == 10
    assert [r[1] for r in mid] == list(range(20))  # event_index in chunk order
    for r in recv:
        c = r[4]
        # start = first slice issued, end = last slice written (+10 ns for slice 1)
        assert r[5] == pytest.approx((1000 * (c + 1)) * 1e-9, abs=2e-9)
        assert r[6] == pytest.approx((1000 * (c + 1) + 510) * 1e-9, abs=2e-9)
        assert r[3] == 0  # peer = predecessor
    tail = chain_rows(rec, lanes, per_lane, plan, n=3, root=0, rank=2)
    assert all(r[2] == "recv" and r[3] == 1 for r in tail)


def test_csv_schema_matches_reference_simulator():
    lanes, per_lane = 4, 3
    plan = {"slices": 2, "slice_bytes": 64, "n_chunks": 4, "ctas": 1}
    rows = []
    for rank in range(2):
        rows += chain_rows(synthetic(lanes, per_lane, plan), lanes, per_lane, plan, n=2, root=0, rank=rank)
    with tempfile.TemporaryDirectory() as d:
        ours = os.path.join(d, "ours.csv")
        write_csv(rows, ours)
        header = open(ours).readline().strip()
        assert header == "rank,event_index,kind,peer,chunk,start_s,end_s"
        if not os.path.exists(HARNESS):
            pytest.skip("oracle/_ref not built here")
        ref = os.path.join(d, "ref.csv")
        subprocess.run([HARNESS, "simulate", "chain_pipelined", "2", "0", "256", "64", "0", "1e-6", "1e9", ref],
                       check=True, capture_output=True)
        assert open(ref).readline().strip() == header
        ref_kinds = {line.split(",")[2] for line in open(ref).read().splitlines()[1:]}
        assert ref_kinds <= {"send", "recv"}
