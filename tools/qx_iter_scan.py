"""Per-codeword vs per-iteration cost of the on-chip exact decoder: fixed
iterations 1..20 (and early stop) on the same config-2 LLRs, CUDA events.
    python tools/qx_iter_scan.py [--k 8448 --n 16896 --m 4 --ebno 6 --batch 8192]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2203_11854_b200 as lb  # noqa: E402
from paper_2203_11854_b200 import ldpc as LD  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--batch", type=int, default=8192)
p.add_argument("--k", type=int, default=8448)
p.add_argument("--n", type=int, default=16896)
p.add_argument("--m", type=int, default=4)
p.add_argument("--ebno", type=float, default=6.0)
p.add_argument("--precision", default="exact")
p.add_argument("--lib", default=None, help="load this liblinksim_b200.so instead (A/B of two builds)")
p.add_argument("--iters", default="1,2,5,10,20")
p.add_argument("--reps", type=int, default=1)
p.add_argument("--modes", default="fixed,es")
a = p.parse_args()
if a.lib:
    from paper_2203_11854_b200 import _lib
    _lib.LIB_PATH = os.path.abspath(a.lib)
cfg = lb.SimConfig.from_dict({"code": {"family": "ldpc5g", "k": a.k, "n": a.n, "decoder": {"mode": "fast"}},
                              "modulation": {"kind": "qam", "bits_per_symbol": a.m},
                              "sweep": {"ebno_db": [a.ebno], "batch_size": a.batch}})
pipe = lb.Pipeline(cfg)
payload, llr = pipe._llr(a.ebno, a.batch, lb.RngStream(1, 2))
res = {}
for es in [m == "es" for m in a.modes.split(",")]:
    for it in [int(x) for x in a.iters.split(",")]:
        def run():
            return LD.qc_decode(llr, pipe.ldpc, it, "min-sum", 0.75, early_stop=es, precision=a.precision,
                                ref_bits=payload, want_hard=False, want_iters=es)
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            r = run()
        e1.record()
        torch.cuda.synchronize()
        key = f"{'es' if es else 'fixed'}_{it}"
        res[key] = {"ms": e0.elapsed_time(e1) / a.reps}
        if es:
            res[key]["mean_iters"] = float(r["iters"].float().mean())
        print(key, res[key], flush=True)
print(json.dumps(res))
