"""C4: PageRank x20 then the triangle count back to back on one lane, against
pagerank_and_triangles (the two on separate library lanes / streams)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1503_07881_b200 as gt  # noqa: E402
from paper_1503_07881_b200.algorithms import pagerank_and_triangles  # noqa: E402
from paper_1503_07881_b200.synth import CONFIGS, rmat_device  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
src, dst = rmat_device(CONFIGS[cfg])
g = gt.table_to_graph(gt.edge_table(src, dst), gt.EdgeSpec("src", "dst"))
del src, dst
out = torch.empty(g.node_count, dtype=torch.float64, device="cuda")
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    gt.pagerank_device(g, 0.85, 20, out.data_ptr())
    tc = gt.triangle_count(g)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    _, tc2 = pagerank_and_triangles(g, 0.85, 20, scores_out_ptr=out.data_ptr())
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"rep {rep}: sequential {1e3*(t1-t0):.1f} ms  two lanes {1e3*(t2-t1):.1f} ms  "
          f"triangles {tc} {tc2} sum={float(out.sum()):.12f}", flush=True)
