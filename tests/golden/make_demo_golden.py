"""Mint tests/golden/demo_waterfall.json: the reference's demos/ldpc_waterfall.py
(Listing-1 sweep: k=500 n=1000 sum-product, 16-QAM max-log, 3-7 dB) run
through the reference's own run_sweep, so the GPU run_sweep of the same
config can be compared point by point (tests/test_gpu_demos.py).

    python tests/golden/make_demo_golden.py   # needs /root/reference
"""
import json
import os
import sys

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
from linksim import SimConfig, run_sweep  # noqa: E402

CONFIG = {
    "code": {"family": "ldpc5g", "k": 500, "n": 1000, "decoder": {"variant": "sum-product", "num_iter": 20}},
    "modulation": {"kind": "qam", "bits_per_symbol": 4, "demapper": "maxlog"},
    "channel": {"kind": "awgn"},
    "sweep": {"ebno_db": [3.0, 4.0, 5.0, 6.0, 7.0], "batch_size": 256, "target_block_errors": 50,
              "max_batches_per_point": 4},
    "seed": 7,
    "precision": "single",
}


def main():
    res = run_sweep(SimConfig.from_dict(CONFIG), num_workers=4)
    pts = [{"ebno_db": p.ebno_db, "bits": p.bits, "bit_errors": p.bit_errors, "blocks": p.blocks,
            "block_errors": p.block_errors, "batches": p.batches, "stop_reason": p.stop_reason}
           for p in res.points]
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "demo_waterfall.json")
    with open(out, "w") as f:
        json.dump({"config": CONFIG, "points": pts}, f, indent=1)
    print(json.dumps(pts))


if __name__ == "__main__":
    main()
