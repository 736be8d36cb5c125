"""Small launches of the on-chip decoders for compute-sanitizer
(racecheck / synccheck / memcheck; one tool per run):

    compute-sanitizer --tool racecheck python tools/sanitize_run.py

Covers the persistent fp16x2 fixed-iteration (k_qc_fast_h2w) and early-stop
slot-refilling (k_qc_fast_h2pw) kernels, the sum-product kernel (k_qc_sp),
and the exact / fp32 full-graph decoder (k_qc_exact, fixed and early stop,
with and without the posterior output)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2203_11854_b200 as lb  # noqa: E402

cfg = lb.SimConfig.from_dict({"code": {"family": "ldpc5g", "k": 8448, "n": 16896, "decoder": {"mode": "fast"}},
                              "modulation": {"kind": "qam", "bits_per_symbol": 4},
                              "sweep": {"ebno_db": [5.0], "batch_size": 8}})
pipe = lb.Pipeline(cfg)
code = pipe.ldpc
iters = int(os.environ.get("SAN_ITERS", "4"))
for ebno in (4.6, 6.5):  # slots converge at different iterations at the lower point
    payload, llr = pipe._llr(ebno, 8, lb.RngStream(3, int(ebno * 10)))
    lb.qc_decode(llr[:4], code, iters, "min-sum", early_stop=False, ref_bits=payload[:4], precision="fp16x2")
    lb.qc_decode(llr, code, 8, "min-sum", early_stop=True, ref_bits=payload, precision="fp16x2", want_iters=True)
    lb.qc_decode(llr[:2], code, iters, "sum-product", early_stop=False, ref_bits=payload[:2])
    for prec in ("exact", "fp32-full"):
        lb.qc_decode(llr[:2], code, iters, "min-sum", early_stop=False, ref_bits=payload[:2], precision=prec)
        lb.qc_decode(llr[:3], code, 8, "scaled-min-sum", early_stop=True, ref_bits=payload[:3], precision=prec,
                     want_llr=True, want_iters=True)
torch.cuda.synchronize()
print("sanitize run done")
