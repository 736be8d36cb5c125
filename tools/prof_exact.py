"""Exact-mode (reference arithmetic) decoder throughput for each BP variant on
config-2 LLRs: python tools/prof_exact.py [--batch 1024] [--early-stop]."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2203_11854_b200 as lb  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--batch", type=int, default=1024)
p.add_argument("--k", type=int, default=8448)
p.add_argument("--n", type=int, default=16896)
p.add_argument("--ebno", type=float, default=6.0)
p.add_argument("--early-stop", action="store_true")
a = p.parse_args()
cfg = lb.SimConfig.from_dict({"code": {"family": "ldpc5g", "k": a.k, "n": a.n, "decoder": {"mode": "fast"}},
                              "modulation": {"kind": "qam", "bits_per_symbol": 4},
                              "sweep": {"ebno_db": [a.ebno], "batch_size": a.batch}})
pipe = lb.Pipeline(cfg)
_, llr = pipe._llr(a.ebno, a.batch, lb.RngStream(1, 2))
for variant in ("min-sum", "scaled-min-sum", "sum-product"):
    for _ in range(2):
        lb.ldpc5g_decode(llr, pipe.ldpc, 20, variant, mode="exact", early_stop=a.early_stop, device=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    lb.ldpc5g_decode(llr, pipe.ldpc, 20, variant, mode="exact", early_stop=a.early_stop, device=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{variant:15s} batch {a.batch} early_stop={a.early_stop}: {ms:8.2f} ms, "
          f"{a.batch * a.k / ms / 1e6:.3f} Gbit/s")
