"""Fast sum-product (k_qc_sp: fp16 messages, product-domain check update) vs
the exact sum-product decoder (CSR engine, the reference's arithmetic) on the
codewords the reference converges on: LLR agreement statistics.

    python tools/sp_accuracy.py [--k 4096 --n 8192 --m 2 --ebno 2.0]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2203_11854_b200 as lb  # noqa: E402
from paper_2203_11854_b200 import ldpc as LD  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--k", type=int, default=4096)
p.add_argument("--n", type=int, default=8192)
p.add_argument("--m", type=int, default=2)
p.add_argument("--ebno", type=float, default=2.0)
p.add_argument("--batch", type=int, default=256)
p.add_argument("--precision", default="fp32", help="fp32 = k_qc_sp (fp16 messages), fp32-full = k_qc_sp32")
a = p.parse_args()
cfg = lb.SimConfig.from_dict({"code": {"family": "ldpc5g", "k": a.k, "n": a.n},
                              "modulation": {"kind": "qam", "bits_per_symbol": a.m},
                              "sweep": {"ebno_db": [a.ebno], "batch_size": a.batch}})
pipe = lb.Pipeline(cfg)
code = pipe.ldpc
payload, llr = pipe._llr(a.ebno, a.batch, lb.RngStream(3, 4))
mother = code.derate_match(llr, device=True)
lo_e, hard_e, it_e = lb.bp_decode(mother, code.pcm, 20, "sum-product", 0.75, True, return_iters=True,
                                  engine="csr", device=True)
r = LD.qc_decode(llr, code, 20, "sum-product", early_stop=True, want_llr=True, want_iters=True,
                 precision=a.precision, prune=True)
# the pruned dead extension rows' parity posteriors are channel values: compare
# the systematic, core-parity and live extension columns
R = lb.ldpc.L.lib().ls_qc_live_rows(code.handle)
ncol = code._kb + max(R, 4)
le, lf = lo_e.cpu().numpy()[:, : ncol * code.z], r["llr"].cpu().numpy()[:, : ncol * code.z]
ie, i_f = it_e.cpu().numpy(), r["iters"].cpu().numpy()
conv = (ie < 20) & (ie == i_f)
d = np.abs(le[conv] - lf[conv]) / np.maximum(np.abs(le[conv]), 1.0)
big = np.abs(le[conv]) > 12.0
res = {"k": a.k, "n": a.n, "ebno": a.ebno, "precision": a.precision, "converged_same_iter": int(conv.sum()),
       "frac_within_1e-4": float((d <= 1e-4).mean()), "frac_within_1e-2": float((d <= 1e-2).mean()),
       "max_rel": float(d.max()), "max_rel_small_llr(|L|<=12)": float(d[~big].max()) if (~big).any() else None,
       "max_rel_large_llr(|L|>12)": float(d[big].max()) if big.any() else None,
       "hard_equal_on_converged": bool(np.array_equal(hard_e.cpu().numpy()[conv][:, :a.k],
                                                      r["hard"].cpu().numpy()[conv]))}
print(json.dumps(res))
