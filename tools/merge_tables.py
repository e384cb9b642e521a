#!/usr/bin/env python3
"""Merge per-n measured tables into one (entries sorted by (n, msg_min)),
validated by the product loader; writes the builtin B200 table."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1707_09414_b200 as B
out, inputs = sys.argv[1], sys.argv[2:]
rows, prov, push = [], [], []
for p in inputs:
    t = B.load_table(p)
    assert t.oracle == "measured", p
    text = open(p).read().splitlines()
    prov.append(text[0][len("# bcl-oracle: measured "):])
    push += [l for l in text[1:] if l.startswith(("# bcl-push-from:", "# bcl-ll128-upto:"))]
    rows += [l for l in text[1:] if l.strip() and not l.startswith("#") and not l.startswith("n,")]
rows.sort(key=lambda l: (int(l.split(",")[0]), int(l.split(",")[1])))
# the library's writer order: push rules, then LL128 rules (each by n)
push.sort(key=lambda l: (not l.startswith("# bcl-push-from:"), int(l.split("n=")[1].split()[0])))
header = "# bcl-oracle: measured " + " | ".join(prov) + "".join("\n" + l for l in push)
text = header + "\nn,msg_min_bytes,msg_max_bytes,algorithm,radix,chunk_bytes,predicted_cost_s\n" + "\n".join(rows) + "\n"
B.load_table_text(text)  # validates ordering / disjoint ranges
open(out, "w").write(text)
print(f"wrote {out}: {len(rows)} entries")
