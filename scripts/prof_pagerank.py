"""PageRank x20 on a BASELINE config's graph, twice (warm-up + measured):
per-phase device times (CUDA events on the library stream)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1503_07881_b200 as gt  # noqa: E402
from paper_1503_07881_b200 import _native  # noqa: E402
from paper_1503_07881_b200.synth import CONFIGS, rmat_device  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
src, dst = rmat_device(CONFIGS[cfg])
g = gt.table_to_graph(gt.edge_table(src, dst), gt.EdgeSpec("src", "dst"))
del src, dst
out = torch.empty(g.node_count, dtype=torch.float64, device="cuda")
for i in range(reps):
    _native.profile_reset()
    _native.profile_enable(True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    gt.pagerank_device(g, 0.85, 20, out.data_ptr())
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    ph = _native.profile_read()
    _native.profile_enable(False)
    e, n = g.edge_count, g.node_count
    it = sum(v[0] for k, v in ph.items() if k in ("pr.spmv", "pr.fixup", "pr.finalize"))
    print(f"rep {i}: pagerank x20 {dt*1e3:.1f} ms  N={n} E={e}  iterations {it:.1f} ms "
          f"-> {(12*e + 32*n) * 20 / (it/1e3) / 1e9:.0f} GB/s (12E+32N)  sum={float(out.sum()):.12f}",
          flush=True)
    for k, (ms, cnt, by) in sorted(ph.items(), key=lambda kv: -kv[1][0]):
        print(f"   {k:24s} {ms:8.2f} ms  x{cnt}  {by/ms/1e6 if ms > 0 else 0:8.1f} GB/s", flush=True)
