"""Where the C4 end-to-end step spends its time: the bench's e2e step (pipelined
prefetch) with the host wall time of each part and the library phase times."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1503_07881_b200 as gt  # noqa: E402
from paper_1503_07881_b200 import _native  # noqa: E402
from paper_1503_07881_b200.synth import CONFIGS, rmat_device  # noqa: E402

spec = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
src, dst = rmat_device(spec)
rows = spec.rows
h_src = torch.empty(rows, dtype=torch.int64, pin_memory=True)
h_dst = torch.empty(rows, dtype=torch.int64, pin_memory=True)
h_src.copy_(src)
h_dst.copy_(dst)
del src, dst
torch.cuda.empty_cache()
host = gt.edge_table(h_src.numpy(), h_dst.numpy())
spec_e = gt.EdgeSpec("src", "dst")
pipe = {"next": None}
d_sc = None
h_sc = None
for it in range(5):
    torch.cuda.synchronize()
    _native.profile_reset()
    _native.profile_enable(True)
    t0 = time.perf_counter()
    cur = pipe["next"] if pipe["next"] is not None else host.prefetch()
    if os.environ.get("PREFETCH_AT") == "start":
        pipe["next"] = host.prefetch()
    g = gt.table_to_graph(cur, spec_e)
    del cur
    t1 = time.perf_counter()
    late = os.environ.get("PREFETCH_AT") == "tc"
    if not late and os.environ.get("PREFETCH_AT") != "start":
        pipe["next"] = host.prefetch()
    t2 = time.perf_counter()
    if d_sc is None:
        d_sc = torch.empty(g.node_count, dtype=torch.float64, device="cuda")
        h_sc = torch.empty(g.node_count, dtype=torch.float64, pin_memory=True)
    gt.pagerank_device(g, 0.85, 20, d_sc.data_ptr())
    if late:
        pipe["next"] = host.prefetch()
    t3 = time.perf_counter()
    tc = gt.triangle_count(g)
    t4 = time.perf_counter()
    h_sc.copy_(d_sc)
    t5 = time.perf_counter()
    ph = _native.profile_read()
    _native.profile_enable(False)
    grp = {}
    for k, (ms, c, b) in ph.items():
        grp[k.split(".")[0]] = grp.get(k.split(".")[0], 0) + ms
    print(f"step {it}: total {1e3*(t5-t0):.1f} ms | build {1e3*(t1-t0):.1f} prefetch-issue {1e3*(t2-t1):.1f} "
          f"pr {1e3*(t3-t2):.1f} tc {1e3*(t4-t3):.1f} d2h {1e3*(t5-t4):.1f} | device phases "
          + " ".join(f"{k} {v:.1f}" for k, v in grp.items()), flush=True)
    del g
