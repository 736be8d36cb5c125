"""fp32 full-graph decoder vs the exact decoder on converged codewords: LLR agreement statistics."""
import sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2203_11854_b200 as lb
from paper_2203_11854_b200 import ldpc as LD
from oracle import linksim_oracle as O


def _llrs(k, n, m, ebno, B, seed):
    oc = O.code(k, n)
    bits = O.binary_source((B, k), seed, 1)
    pts = O.qam_points(m)
    x = O.map_bits(oc.encode(bits), pts, m).astype(np.complex64)
    no = O.ebnodb2no(ebno, m, k / n)
    y = O.awgn_single(x, no, seed, 2)
    return bits, O.demap(y, no, pts, m).astype(np.float32)
for (k, n, m, ebno) in [(256, 512, 2, 3.0), (256, 512, 2, 3.5), (256, 512, 2, 4.0), (8448, 16896, 4, 5.8), (4096, 12288, 6, 7.6)]:
    code = lb.LdpcCode5G(k, n)
    B = 64 if k > 4000 else 256
    bits, llr = _llrs(k, n, m, ebno, B, 21)
    for variant in ("min-sum", "scaled-min-sum"):
        ex = LD.qc_decode(llr, code, 20, variant, 0.75, early_stop=True, precision="exact", want_llr=True, want_iters=True)
        f = LD.qc_decode(llr, code, 20, variant, 0.75, early_stop=True, precision="fp32-full", want_llr=True, want_iters=True)
        ie, i_f = ex["iters"].cpu().numpy(), f["iters"].cpu().numpy()
        conv = ie < 20
        same = conv & (ie == i_f)
        le, lf = ex["llr"].cpu().numpy()[same], f["llr"].cpu().numpy()[same]
        d = np.abs(le - lf) / np.maximum(np.abs(le), 1.0)
        rowbad = (d > 1e-4).any(axis=1)
        print(k, n, ebno, variant, "conv", conv.sum(), "same_it", same.sum(), "frac<=1e-4 %.5f" % (d <= 1e-4).mean(),
              "max %.2e" % d.max(), "rows with any >1e-4:", rowbad.sum(), "hard eq", np.array_equal(ex["hard"].cpu().numpy()[conv], f["hard"].cpu().numpy()[conv]))
