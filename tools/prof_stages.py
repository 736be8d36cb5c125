"""Per-stage CUDA-event timing of one Pipeline batch (config 2 by default)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2203_11854_b200 as lb  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--batch", type=int, default=65536)
p.add_argument("--k", type=int, default=8448)
p.add_argument("--n", type=int, default=16896)
p.add_argument("--m", type=int, default=4)
p.add_argument("--ebno", type=float, default=6.0)
p.add_argument("--noise", default="philox", choices=["philox", "numpy"])
p.add_argument("--decoder", default="fp16x2", choices=["fp16x2", "fp32", "exact"])
a = p.parse_args()
code = lb.LdpcCode5G(a.k, a.n)
const = lb.Constellation("qam", a.m)
no = lb.ebnodb2no(a.ebno, a.m, a.k / a.n)


def run(timed):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(8)]
    rng = lb.RngStream(1, 2)
    ev[0].record()
    bits = lb.binary_source([a.batch, a.k], rng.child(0), device=True)
    ev[1].record()
    tx = lb.ldpc5g_encode(bits, code, device=True)
    ev[2].record()
    x = lb.map_bits(tx, const, device=True)
    ev[3].record()
    y = lb.awgn(x, no, rng.child(2), device=True, noise=a.noise)
    ev[4].record()
    llr = lb.demap_app(y, no, const, out_dtype="float32", device=True)
    ev[5].record()
    res = lb.qc_decode(llr, code, 20, "min-sum", early_stop=False, ref_bits=bits, want_hard=False,
                       precision=a.decoder)
    ev[6].record()
    torch.cuda.synchronize()
    if timed:
        names = ["source", "encode", "map", "awgn", "demap", "decode"]
        for j, nm in enumerate(names):
            print(f"{nm:8s} {ev[j].elapsed_time(ev[j + 1]):9.3f} ms")
        print("counts", res["counts"].tolist())


run(False)
run(True)
