"""Statistical parity of the GPU config-3 sweep against the CPU oracle
(SURVEY.md 8c tier 3): BLER at waterfall points from profiles/r01/sweep_c3_*.csv
(fast decoder, Philox noise, 8192-codeword batches on the B200) versus the
oracle's run_batch (reference arithmetic, numpy noise) on independent
streams, with 95% Wilson intervals for both.

  python tools/compare_c3.py [--codewords 2048]   (CPU; writes profiles/r01/c3_oracle_check.json)
"""
import argparse
import concurrent.futures
import csv
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import linksim_oracle as O  # noqa: E402


def wilson(k, n, z=1.96):
    if n == 0:
        return (0.0, 1.0)
    p = k / n
    d = 1 + z * z / n
    c = (p + z * z / (2 * n)) / d
    h = z * math.sqrt(p * (1 - p) / n + z * z / (4 * n * n)) / d
    return (max(0.0, c - h), min(1.0, c + h))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--codewords", type=int, default=2048)
    ap.add_argument("--points", default="2.5,3.0")
    a = ap.parse_args()
    out = {"note": __doc__.strip().splitlines()[0], "points": []}
    per = 32
    nb = a.codewords // per
    for variant in ("min-sum", "sum-product"):
        gpu = {float(r["ebno_db"]): r for r in
               csv.DictReader(open(os.path.join(ROOT, "profiles", "r01", f"sweep_c3_{variant}.csv")))}
        for eb in (float(x) for x in a.points.split(",")):
            def one(b):
                p, d = O.run_batch(4096, 8192, 2, eb, per, 99, ((b + 1) << 32) | 7, variant)
                return int((p != d).any(axis=1).sum())
            with concurrent.futures.ThreadPoolExecutor(os.cpu_count() or 4) as ex:
                blk = sum(ex.map(one, range(nb)))
            g = gpu[eb]
            gk, gn = int(g["block_errors"]), int(g["blocks"])
            lo_o, hi_o = wilson(blk, nb * per)
            lo_g, hi_g = wilson(gk, gn)
            out["points"].append({
                "variant": variant, "ebno_db": eb,
                "oracle": {"blocks": nb * per, "block_errors": blk, "bler": blk / (nb * per), "ci95": [lo_o, hi_o]},
                "gpu_fast": {"blocks": gn, "block_errors": gk, "bler": gk / gn, "ci95": [lo_g, hi_g]},
                "intervals_overlap": not (hi_o < lo_g or hi_g < lo_o)})
            print(out["points"][-1], flush=True)
    with open(os.path.join(ROOT, "profiles", "r01", "c3_oracle_check.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
