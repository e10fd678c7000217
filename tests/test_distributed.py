"""Multi-process path (distributed.py) on CPU: gloo, world size 2, 3 and 4.

Drives the real orchestration — id-range and presence all-reduces, splitter
histograms, the two all-to-all shuffles, offset rebasing, PageRank's
per-iteration all-gather / all-reduce, the triangle all-reduce — with the CPU
restatement of the per-rank primitives (dist_cpu_ops.CpuOps), and checks the
result against the oracle (the reference restated, pinned to its goldens).
The same orchestration runs over NCCL with NativeOps on the GPU
(test_distributed_gpu.py).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import reference_port as ref

TIMEOUT_S = 180


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case_file, out_file, cuts):
    import sys
    from pathlib import Path

    repo = Path(__file__).resolve().parent.parent
    for p in (str(repo), str(repo / "tests")):
        if p not in sys.path:
            sys.path.insert(0, p)
    import torch.distributed as dist

    from dist_cpu_ops import CpuOps
    from paper_1503_07881_b200 import distributed as D

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        data = np.load(case_file)
        a, b = cuts[rank], cuts[rank + 1]
        src = torch.from_numpy(data["src"][a:b].copy())
        dst = torch.from_numpy(data["dst"][a:b].copy())
        ops = CpuOps()
        sg = D.build_csr(src, dst, ops=ops)
        out_off, out_adj, in_off, in_adj = D.gather_csr(sg)
        pr = D.pagerank(sg, 0.85, 10, ops=ops) if sg.n else torch.zeros(0, dtype=torch.float64)
        tc = D.triangle_count(sg, ops=ops)
        if rank == 0:
            np.savez(out_file, n=sg.n, e=sg.e, ids=sg.ids.numpy(), out_off=out_off.numpy(),
                     out_adj=out_adj.numpy(), in_off=in_off.numpy(), in_adj=in_adj.numpy(),
                     pr=pr.numpy(), tc=tc, out_bounds=np.asarray(sg.out_bounds),
                     in_bounds=np.asarray(sg.in_bounds))
    finally:
        dist.destroy_process_group()


def _run(tmp_path, src, dst, world, cuts=None):
    rows = src.shape[0]
    if cuts is None:
        cuts = [rows * r // world for r in range(world + 1)]
    case = tmp_path / "case.npz"
    out = tmp_path / "out.npz"
    np.savez(case, src=src.astype(np.int64), dst=dst.astype(np.int64))
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, str(case), str(out), cuts))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(TIMEOUT_S)
    for p in procs:
        if p.is_alive():
            p.kill()
            pytest.fail("distributed worker timed out")
        assert p.exitcode == 0, f"worker exit code {p.exitcode}"
    return np.load(out)


def _check(res, src, dst):
    want = ref.build_csr(src.astype(np.int64), dst.astype(np.int64), workers=1)
    assert int(res["n"]) == want.n and int(res["e"]) == want.e
    ids = res["ids"]
    assert np.array_equal(ids, want.ids)
    assert np.array_equal(res["out_off"], want.out_off)
    assert np.array_equal(res["in_off"], want.in_off)
    assert np.array_equal(ids[res["out_adj"]], want.out_adj)
    assert np.array_equal(ids[res["in_adj"]], want.in_adj)
    if want.n:
        pr_want = ref.pagerank_csr(want, 0.85, 10, workers=1)
        assert float(np.abs(res["pr"] - pr_want).sum()) <= 1e-9
    assert int(res["tc"]) == ref.triangle_count_fast(want)
    # the ranges tile the node set
    for b in (res["out_bounds"], res["in_bounds"]):
        assert b[0] == 0 and b[-1] == want.n and np.all(np.diff(b) >= 0)


def test_two_ranks_random_table_with_duplicates_negatives_selfloops(tmp_path):
    rng = np.random.default_rng(21)
    src = rng.integers(-40, 260, size=3000)
    dst = rng.integers(-40, 260, size=3000)
    src[:50] = dst[:50]  # self-loops
    src = np.concatenate([src, src[:400]])  # duplicate rows across the split
    dst = np.concatenate([dst, dst[:400]])
    _check(_run(tmp_path, src, dst, 2), src, dst)


def test_three_ranks_skewed_rmat(tmp_path):
    from paper_1503_07881_b200.synth import rmat_edges

    src, dst = rmat_edges(9, 6000, seed=5)
    _check(_run(tmp_path, src, dst, 3), src, dst)


def test_two_ranks_one_empty_slice(tmp_path):
    from paper_1503_07881_b200.synth import rmat_edges

    src, dst = rmat_edges(8, 2500, seed=6, permute=True)
    _check(_run(tmp_path, src, dst, 2, cuts=[0, 0, src.shape[0]]), src, dst)


def test_two_ranks_empty_table(tmp_path):
    src = np.zeros(0, dtype=np.int64)
    res = _run(tmp_path, src, src, 2)
    assert int(res["n"]) == 0 and int(res["e"]) == 0 and int(res["tc"]) == 0


def test_four_ranks_rmat_with_hubs(tmp_path):
    """World size 4, uneven slices: PageRank's padded all-gather layout with
    unequal dst ranges, the shuffles, the triangle split."""
    from paper_1503_07881_b200.synth import rmat_edges

    src, dst = rmat_edges(10, 9000, seed=8, permute=True)
    cuts = [0, 1000, 4000, 4100, src.shape[0]]
    _check(_run(tmp_path, src, dst, 4, cuts=cuts), src, dst)
