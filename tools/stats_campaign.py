"""Statistical parity of the fast decoders at scale: block-error outcomes of
every fast decoder against the reference's own (the exact decoder for the
min-sum variants, bit-identical to the reference; the f64 CSR engine for
sum-product) on the same exact-chain LLRs (numpy-exact noise, f64
demapper), over waterfall Eb/N0 points of configs 2 and 3.  Reports BLER,
the two-proportion z and the McNemar z of the paired outcomes.

    python tools/stats_campaign.py [--scale 1.0] > profiles/r02/stats_campaign.json
"""
import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2203_11854_b200 as lb  # noqa: E402
from paper_2203_11854_b200 import ldpc as LD  # noqa: E402

# (k, n, bits per symbol, Eb/N0 points, codewords per point)
CASES = [
    (8448, 16896, 4, [4.4, 4.6, 4.8, 5.0, 5.4, 5.6, 5.8], 32768),
    (4096, 8192, 2, [1.25, 1.5, 1.75, 2.0, 2.25, 2.5, 2.75, 3.0], 65536),
]
# (variant, reference precision, fast precisions)
DECODERS = [
    ("min-sum", "exact", ["fp16x2", "fp32-full"]),
    ("scaled-min-sum", "exact", ["fp16x2", "fp32-full"]),
    ("sum-product", "csr", ["fp32", "fp32-full"]),
]


def _block_errors(llr, code, variant, precision, payload, chunk):
    out = []
    for lo in range(0, llr.shape[0], chunk):
        x = llr[lo:lo + chunk]
        if precision == "csr":  # the reference's sum-product arithmetic (f64 CSR engine)
            mother = code.derate_match(x, device=True)
            _, hard = lb.bp_decode(mother, code.pcm, 20, variant, 0.75, True, engine="csr", device=True)
            hard = hard[:, : code.k]
        else:
            hard = LD.qc_decode(x, code, 20, variant, 0.75, early_stop=True, precision=precision)["hard"]
        out.append((hard != payload[lo:lo + chunk]).any(dim=1))
    return torch.cat(out)


def _stats(ref, fast):
    n = ref.numel()
    a, b = int(ref.sum()), int(fast.sum())
    n10 = int((ref & ~fast).sum())  # reference fails, fast decodes
    n01 = int((~ref & fast).sum())
    p = (a + b) / (2 * n)
    z2 = (b - a) / n / math.sqrt(max(2 * p * (1 - p) / n, 1e-300)) if 0 < p < 1 else 0.0
    zm = (n01 - n10) / math.sqrt(n01 + n10) if n01 + n10 else 0.0
    return {"blocks": n, "ref_block_errors": a, "block_errors": b, "discordant_ref_fails_only": n10,
            "discordant_fast_fails_only": n01, "two_proportion_z": round(z2, 3), "mcnemar_z": round(zm, 3)}


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--scale", type=float, default=1.0)
    a = p.parse_args()
    res = []
    for k, n, m, points, B in CASES:
        B = max(64, int(B * a.scale))
        cfg = lb.SimConfig.from_dict({"code": {"family": "ldpc5g", "k": k, "n": n},
                                      "modulation": {"kind": "qam", "bits_per_symbol": m},
                                      "sweep": {"ebno_db": points, "batch_size": B}})
        pipe = lb.Pipeline(cfg)
        code = pipe.ldpc
        for ebno in points:
            payload, llr = pipe._llr(ebno, B, lb.RngStream(11, (k << 12) ^ int(ebno * 1000)))
            for variant, refp, fasts in DECODERS:
                chunk = 4096 if refp == "csr" else B
                ref = _block_errors(llr, code, variant, refp, payload, chunk)
                for fp in fasts:
                    if not LD.qc_has_kernel(code, precision=fp, variant=variant):
                        continue
                    fast = _block_errors(llr, code, variant, fp, payload, B)
                    rec = {"k": k, "n": n, "ebno_db": ebno, "variant": variant, "reference": refp,
                           "fast": fp, **_stats(ref, fast)}
                    res.append(rec)
                    print(json.dumps(rec), file=sys.stderr, flush=True)
    worst = max(abs(r["two_proportion_z"]) for r in res)
    print(json.dumps({"points": res, "max_abs_two_proportion_z": worst,
                      "all_within_3_sigma": worst < 3.0}, indent=1))


if __name__ == "__main__":
    main()
