"""Receive side of the sharded build: gt_merge_runs vs re-sorting the
concatenated runs (gt_sort_keys over the full key / over the dst bits)."""
import sys

import numpy as np
import torch

from paper_1503_07881_b200.distributed import NativeOps


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    ops = NativeOps("cuda:0")
    total = int(sys.argv[1]) if len(sys.argv) > 1 else 128_000_000
    kbits = 24
    for nruns in (2, 4, 8):
        per = total // nruns
        g = torch.Generator(device="cuda").manual_seed(nruns)
        keys = torch.randint(0, 1 << (2 * kbits), (per * nruns,), device="cuda", generator=g)
        runs = keys.view(nruns, per).sort(dim=1).values.reshape(-1).contiguous()
        sizes = [per] * nruns
        tm = timed(lambda: ops.merge_runs(runs, sizes))
        ts = timed(lambda: ops.sort_keys(runs, 0, 2 * kbits))
        td = timed(lambda: ops.sort_keys(runs, kbits, 2 * kbits))
        gb = runs.numel() * 8 / 1e9
        print(f"runs={nruns} keys={runs.numel()} merge {tm:.2f} ms "
              f"({gb * 2 * int(np.ceil(np.log2(nruns))) / tm * 1e3:.0f} GB/s algorithmic) | "
              f"sort 0..{2*kbits} {ts:.2f} ms | sort dst bits {td:.2f} ms "
              f"(both include one clone of the input)")
        del keys, runs


if __name__ == "__main__":
    main()
