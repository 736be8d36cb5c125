"""Timing of the numpy-exact normal generator (ls_standard_normal) and the
exact awgn, per call after warm-up."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2203_11854_b200 as lb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 553_000_000
for i in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    z = lb.channel.standard_normal(n, lb.RngStream(1, 2 + i), device=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"standard_normal {n}: {dt * 1e3:.1f} ms  ({n / dt / 1e9:.2f} G normals/s)")
    del z
