"""L2 throughput of this B200 for the gather-form sparse kernels (K8 / K9):
streaming an L2-resident buffer, and random row gathers of r doubles (lanes
over the row) -- the access pattern of mc_sampled_k (U rows, r = 50 at C4) and
csr_spmm_k (X rows, b ~ 51-61). Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1012_0365_b200 as B  # noqa: E402

ctx = B.Context(0)
out = {"l2_stream_GBps": round(ctx.l2_probe(0), 1)}
for row in (32, 50, 55, 64, 100):
    out[f"gather_row{row}_GBps"] = round(ctx.l2_probe(1, row), 1)
print(json.dumps(out), flush=True)
