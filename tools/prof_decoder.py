"""Decoder-only driver for ncu captures: prepares a batch of config-2 LLRs on
the GPU, then launches the fast QC decoder `--reps` times.

  python tools/prof_decoder.py --batch 2048 --reps 3
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2203_11854_b200 as lb  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--batch", type=int, default=2048)
p.add_argument("--reps", type=int, default=3)
p.add_argument("--k", type=int, default=8448)
p.add_argument("--n", type=int, default=16896)
p.add_argument("--m", type=int, default=4)
p.add_argument("--ebno", type=float, default=6.0)
p.add_argument("--iters", type=int, default=20)
p.add_argument("--variant", default="min-sum")
p.add_argument("--early-stop", action="store_true")
p.add_argument("--precision", default="fp32")
a = p.parse_args()
cfg = lb.SimConfig.from_dict({"code": {"family": "ldpc5g", "k": a.k, "n": a.n},
                              "modulation": {"kind": "qam", "bits_per_symbol": a.m},
                              "sweep": {"ebno_db": [a.ebno], "batch_size": a.batch}})
pipe = lb.Pipeline(cfg)
payload, llr = pipe._llr(a.ebno, a.batch, lb.RngStream(1, 2))
counts = torch.zeros(2, dtype=torch.int64, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for r in range(a.reps):
    if r == a.reps - 1:
        ev[0].record()
    lb.qc_decode(llr, pipe.ldpc, a.iters, a.variant, early_stop=a.early_stop, ref_bits=payload,
                 want_hard=False, counts=counts, precision=a.precision)
ev[1].record()
torch.cuda.synchronize()
ms = ev[0].elapsed_time(ev[1])
print(f"batch {a.batch} iters {a.iters}: {ms:.3f} ms/launch, "
      f"{a.batch * a.k / ms / 1e6:.3f} Gbit/s, counts summed over {a.reps} launches {counts.tolist()}")
