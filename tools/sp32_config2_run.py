import os, sys, torch; sys.path.insert(0, "/root/repo")
if len(sys.argv) > 1:
    from paper_2203_11854_b200 import _lib
    _lib.LIB_PATH = os.path.abspath(sys.argv[1])
import paper_2203_11854_b200 as lb
B = 8192
pipe = lb.Pipeline(lb.SimConfig.from_dict({"code": {"family": "ldpc5g", "k": 8448, "n": 16896, "decoder": {"mode": "fast"}},
    "modulation": {"kind": "qam", "bits_per_symbol": 4}, "sweep": {"ebno_db": [4.8], "batch_size": B}}))
payload, llr = pipe._llr(4.8, B, lb.RngStream(3, 31))
for prec in ("fp32-full", "fp32"):
    def run():
        return lb.qc_decode(llr, pipe.ldpc, 20, "sum-product", early_stop=False, ref_bits=payload, want_hard=False, precision=prec)
    run(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); r = run(); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1); print(prec, ms, B * 8448 / ms / 1e6, r["counts"].tolist())
