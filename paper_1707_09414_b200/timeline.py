"""Device timelines in the reference's trace CSV schema.

The reference simulator writes `rank,event_index,kind,peer,chunk,start_s,end_s`
(proj/src/simengine.cpp:295-305). `Comm.set_trace` makes every lane of the
device executor stamp %globaltimer per pull; `chain_rows` folds those per-slice
records into one recv event per (rank, chunk) — start = first slice issued,
end = last slice written — plus the forwarding send of interior ranks, so a
measured B200 broadcast and a reference simulation can be diffed row by row.
Times are seconds from the rank's own kernel start (GPU clocks are not
synchronised across devices).
"""
from typing import List, Sequence


def trace_words(lanes: int, per_lane: int) -> int:
    """int64 words to allocate for `Comm.set_trace(records, per_lane)`."""
    return lanes * per_lane * 4


def chain_rows(records, lanes: int, per_lane: int, plan: dict, n: int, root: int, rank: int) -> List[list]:
    """Rows for one rank of a chain_pipelined broadcast.

    records: the rank's trace buffer (CPU int64 tensor/array of trace_words)."""
    import numpy as np
    rec = np.asarray(records, dtype=np.int64).reshape(lanes, per_lane, 4)
    life = rec[:, per_lane - 1, :]
    active = life[:, 0] > 0
    t0 = int(life[active, 0].min()) if active.any() else 0
    q, k_chunks = plan["slices"], plan["n_chunks"]
    ns = lanes // q
    logical = (rank - root) % n
    prev, nxt = (rank - 1) % n, (rank + 1) % n
    rows = []
    if logical == 0:  # the head publishes every chunk at kernel start
        for c in range(k_chunks):
            rows.append([rank, c, "send", nxt, c, 0.0, 0.0])
        return rows
    start = np.full(k_chunks, np.iinfo(np.int64).max, dtype=np.int64)
    end = np.zeros(k_chunks, dtype=np.int64)
    for lane in range(min(lanes, ns * q)):
        pipe = lane // q
        for k in range(per_lane - 1):
            r = rec[lane, k]
            if r[0] == 0 and r[2] == 0:
                continue
            c = pipe + k * ns
            if c >= k_chunks:
                break
            begin = r[0] if r[0] else r[1]
            done = max(r[2], r[1])
            start[c] = min(start[c], begin)
            end[c] = max(end[c], done)
    idx = 0
    for c in range(k_chunks):
        if end[c] == 0:
            continue
        s, e = (start[c] - t0) * 1e-9, (end[c] - t0) * 1e-9
        rows.append([rank, idx, "recv", prev, c, s, e])
        idx += 1
        if logical < n - 1:
            rows.append([rank, idx, "send", nxt, c, e, e])
            idx += 1
    return rows


def write_csv(rows: Sequence[list], path: str) -> None:
    with open(path, "w") as f:
        f.write("rank,event_index,kind,peer,chunk,start_s,end_s\n")
        for r in sorted(rows, key=lambda x: (x[0], x[1])):
            f.write(f"{r[0]},{r[1]},{r[2]},{r[3]},{r[4]},{r[5]:.9g},{r[6]:.9g}\n")
