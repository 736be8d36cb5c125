"""Pipeline.run_batch (host outputs) at several chunk sizes, config 2 fast
mode: python tools/prof_runbatch.py."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2203_11854_b200 as lb  # noqa: E402

B = 65536
cfg = lb.SimConfig.from_dict({"code": {"family": "ldpc5g", "k": 8448, "n": 16896,
                                       "decoder": {"mode": "fast", "variant": "min-sum", "early_stop": False}},
                              "modulation": {"kind": "qam", "bits_per_symbol": 4},
                              "sweep": {"ebno_db": [6.0], "batch_size": B}})
pipe = lb.Pipeline(cfg)
for chunk in (16384, 8192, 4096, 8192, 32768):
    for i in range(2):
        pipe.run_batch(6.0, B, lb.RngStream(1, 100 + i), chunk=chunk)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for i in range(3):
        pipe.run_batch(6.0, B, lb.RngStream(1, i), chunk=chunk)
    el = (time.perf_counter() - t) / 3
    print(f"chunk {chunk:6d}: {el * 1e3:7.1f} ms/step, {B * 8448 / el / 1e9:.2f} Gbit/s")
