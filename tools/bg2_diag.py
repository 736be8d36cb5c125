import sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2203_11854_b200 as lb
from oracle import linksim_oracle as O
for z in (32, 384):
    k = 10 * z; n = 3 * k
    code = lb.LdpcCode5G(k, n, base_graph=2, z=z); oc = O.Code(k, n, bg=2, z=z)
    for ebno in (1.0, 2.0, 3.0, 4.0, 6.0):
        bits = O.binary_source((16, k), 5, 1)
        pts = O.qam_points(2)
        x = O.map_bits(oc.encode(bits), pts, 2).astype(np.complex64)
        no = O.ebnodb2no(ebno, 2, k / n)
        y = O.awgn_single(x, no, 5, 2)
        llr = O.demap(y, no, pts, 2).astype(np.float32)
        raw = ((llr > 0) != oc.encode(bits)).mean()
        lo, hard, it = lb.bp_decode(oc.derate_match(llr), code.pcm, 20, "min-sum", 0.75, True, return_iters=True)
        ok = (hard[:, :k] == bits).all(axis=1)
        print(z, ebno, "raw BER %.4f" % raw, "iters", it.tolist()[:8], "ok", ok.sum())
