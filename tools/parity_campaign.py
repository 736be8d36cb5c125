"""Bit-identity of the on-chip exact decoder against the oracle at scale
(thousands of codewords per configuration, more than the -m gpu tests run):
GPU `ldpc5g_decode(mode="exact")` / `qc_decode(precision="exact")` on the
exact chain's LLRs (numpy-exact noise, f64 demapper) against the C
restatement of bp_decode (oracle/, itself pinned to reference-minted
goldens), on the GPU box's host cores.  Compares decoded bits, mother
llr_out (bitwise) and per-row iteration counts, with early stop.

    python tools/parity_campaign.py [--scale 1.0] > profiles/r02/parity_campaign.json
"""
import argparse
import concurrent.futures
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2203_11854_b200 as lb  # noqa: E402
from paper_2203_11854_b200 import ldpc as LD  # noqa: E402
from oracle import linksim_oracle as O  # noqa: E402

# (k, n, bits per symbol, Eb/N0 dB, codewords): BASELINE configs 1-4 in and
# around the waterfall, where iteration counts spread the most
CASES = [
    (256, 512, 2, 3.0, 16384), (256, 512, 2, 4.5, 16384),
    (8448, 16896, 4, 5.4, 2048), (8448, 16896, 4, 6.0, 2048),
    (4096, 8192, 2, 2.5, 4096), (4096, 8192, 2, 3.25, 4096),
    (4096, 12288, 6, 7.0, 2048),
]


def oracle_decode(llr, oc, variant, threads, chunk):
    def one(lo):
        return O.decode(llr[lo:lo + chunk], oc, 20, variant, 0.75, True)

    with concurrent.futures.ThreadPoolExecutor(threads) as ex:
        parts = list(ex.map(one, range(0, llr.shape[0], chunk)))
    return (np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts]),
            np.concatenate([p[2] for p in parts]))


# whole exact-mode Pipeline.run_batch (payload, encoder, mapper, numpy-exact
# noise, f64 demapper, exact decoder) against the oracle's run_batch:
# (k, n, bits per symbol, Eb/N0, variant, batches, batch size)
CHAIN_CASES = [
    (256, 512, 2, 3.5, "min-sum", 64, 256),
    (8448, 16896, 4, 5.6, "min-sum", 32, 64),
    (4096, 8192, 2, 3.0, "scaled-min-sum", 32, 128),
    (4096, 12288, 6, 7.5, "min-sum", 32, 64),
]


def chain_campaign(a):
    res = []
    for k, n, m, ebno, variant, nb, bs in CHAIN_CASES:
        nb = max(2, int(nb * a.scale))
        cfg = lb.SimConfig.from_dict({"code": {"family": "ldpc5g", "k": k, "n": n,
                                               "decoder": {"variant": variant, "num_iter": 20}},
                                      "modulation": {"kind": "qam", "bits_per_symbol": m},
                                      "sweep": {"ebno_db": [ebno], "batch_size": bs}})
        pipe = lb.Pipeline(cfg)
        seed = 1000 + k
        gpu = [pipe.run_batch(ebno, bs, lb.RngStream(seed, (1 << 32) | (b + 1))) for b in range(nb)]
        t0 = time.perf_counter()
        with concurrent.futures.ThreadPoolExecutor(a.threads) as ex:
            ref = list(ex.map(lambda b: O.run_batch(k, n, m, ebno, bs, seed, (1 << 32) | (b + 1), variant),
                              range(nb)))
        el = time.perf_counter() - t0
        same_p = sum(int(np.array_equal(g[0], r[0])) for g, r in zip(gpu, ref))
        same_d = sum(int(np.array_equal(g[1], r[1])) for g, r in zip(gpu, ref))
        rec = {"k": k, "n": n, "m": m, "ebno_db": ebno, "variant": variant, "batches": nb, "batch_size": bs,
               "codewords": nb * bs, "identical_payload_batches": same_p, "identical_decoded_batches": same_d,
               "block_errors": int(sum((r[0] != r[1]).any(axis=1).sum() for r in ref)),
               "oracle_seconds": round(el, 1)}
        rec["all_identical"] = same_p == nb and same_d == nb
        res.append(rec)
        print(json.dumps(rec), file=sys.stderr, flush=True)
    return res


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--scale", type=float, default=1.0, help="multiply every case's codeword count")
    p.add_argument("--threads", type=int, default=os.cpu_count() or 8)
    p.add_argument("--chain", action="store_true", help="also compare whole exact-mode run_batch chains")
    a = p.parse_args()
    out = {"threads": a.threads, "cases": []}
    if a.chain:
        out["chain_cases"] = chain_campaign(a)
    for k, n, m, ebno, B in CASES:
        B = max(8, int(B * a.scale))
        cfg = lb.SimConfig.from_dict({"code": {"family": "ldpc5g", "k": k, "n": n},
                                      "modulation": {"kind": "qam", "bits_per_symbol": m},
                                      "sweep": {"ebno_db": [ebno], "batch_size": B}})
        pipe = lb.Pipeline(cfg)
        payload, llr_d = pipe._llr(ebno, B, lb.RngStream(7, (k << 8) ^ int(ebno * 100)))
        llr = llr_d.cpu().numpy()
        oc = O.code(k, n)
        for variant in ("min-sum", "scaled-min-sum"):
            r = LD.qc_decode(llr_d, pipe.ldpc, 20, variant, 0.75, early_stop=True, precision="exact",
                             want_llr=True, want_iters=True)
            g_hard, g_llr, g_it = (r["hard"].cpu().numpy(), r["llr"].cpu().numpy(), r["iters"].cpu().numpy())
            t0 = time.perf_counter()
            o_hard, o_llr, o_it = oracle_decode(llr, oc, variant, a.threads, 4 if k > 4000 else 32)
            el = time.perf_counter() - t0
            same_llr = np.all(g_llr.view(np.uint32) == o_llr.view(np.uint32), axis=1)
            rec = {"k": k, "n": n, "m": m, "ebno_db": ebno, "variant": variant, "codewords": B,
                   "identical_llr_out_rows": int(same_llr.sum()),
                   "identical_hard_rows": int(np.all(g_hard == o_hard, axis=1).sum()),
                   "identical_iters": int((g_it == o_it).sum()),
                   "iters_histogram": {int(u): int(c) for u, c in zip(*np.unique(o_it, return_counts=True))},
                   "block_errors_vs_payload": int(np.any(o_hard != payload.cpu().numpy(), axis=1).sum()),
                   "oracle_seconds": round(el, 1)}
            rec["all_identical"] = (rec["identical_llr_out_rows"] == B and rec["identical_hard_rows"] == B
                                    and rec["identical_iters"] == B)
            out["cases"].append(rec)
            print(json.dumps(rec), file=sys.stderr, flush=True)
    out["all_identical"] = all(c["all_identical"] for c in out["cases"] + out.get("chain_cases", []))
    out["codewords_compared"] = sum(c["codewords"] for c in out["cases"])
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
