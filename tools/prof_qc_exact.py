"""On-chip exact decoder (bp_qc_exact.cuh) throughput on config-2 LLRs, next
to the HBM-streaming CSR exact decoder, with a bit-identity check between
the two: python tools/prof_qc_exact.py [--batch 8192] [--ebno 6.0]."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2203_11854_b200 as lb  # noqa: E402
from paper_2203_11854_b200 import ldpc as LD  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--batch", type=int, default=8192)
p.add_argument("--k", type=int, default=8448)
p.add_argument("--n", type=int, default=16896)
p.add_argument("--m", type=int, default=4)
p.add_argument("--ebno", type=float, default=6.0)
p.add_argument("--reps", type=int, default=3)
p.add_argument("--check", type=int, default=64)
a = p.parse_args()
cfg = lb.SimConfig.from_dict({"code": {"family": "ldpc5g", "k": a.k, "n": a.n, "decoder": {"mode": "fast"}},
                              "modulation": {"kind": "qam", "bits_per_symbol": a.m},
                              "sweep": {"ebno_db": [a.ebno], "batch_size": a.batch}})
pipe = lb.Pipeline(cfg)
code = pipe.ldpc
payload, llr = pipe._llr(a.ebno, a.batch, lb.RngStream(1, 2))
res = {"batch": a.batch, "k": a.k, "n": a.n, "ebno": a.ebno}


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out


for prec, variant, es in (("exact", "min-sum", False), ("exact", "min-sum", True), ("exact", "scaled-min-sum", False),
                          ("exact", "scaled-min-sum", True), ("fp32-full", "min-sum", False),
                          ("fp32-full", "min-sum", True)):
    if True:
        counts = torch.zeros(2, dtype=torch.int64, device="cuda")

        def run():
            counts.zero_()
            return LD.qc_decode(llr, code, 20, variant, 0.75, early_stop=es, precision=prec, ref_bits=payload,
                                want_hard=False, want_iters=es, counts=counts)

        ms, r = timed(run, a.reps)
        key = f"{prec}_{variant}_{'es' if es else 'fixed'}"
        res[key] = {"ms": ms, "gbit_s": a.batch * a.k / ms / 1e6, "counts": counts.tolist()}
        if es:
            res[key]["mean_iters"] = float(r["iters"].float().mean())
        print(key, res[key], flush=True)

# bit identity against the CSR exact engine on a slice
if a.check:
    mother = code.derate_match(llr[: a.check], device=True)
    for variant in ("min-sum", "scaled-min-sum"):
        x = lb.bp_decode(mother, code.pcm, 20, variant, 0.75, True, return_iters=True, engine="qc", device=True)
        y = lb.bp_decode(mother, code.pcm, 20, variant, 0.75, True, return_iters=True, engine="csr", device=True)
        same = all(bool(torch.equal(u.view(torch.int32) if u.dtype == torch.float32 else u,
                                    v.view(torch.int32) if v.dtype == torch.float32 else v)) for u, v in zip(x, y))
        res[f"identical_to_csr_{variant}"] = same
        print(variant, "identical to CSR engine:", same, flush=True)
    torch.cuda.synchronize()
    ms, _ = timed(lambda: lb.bp_decode(mother, code.pcm, 20, "min-sum", 0.75, False, engine="csr", device=True), 1)
    res["csr_fixed_min_sum_gbit_s"] = a.check * a.k / ms / 1e6
print(json.dumps(res))
