"""GPU measurements for BASELINE.json configs 3-5 (one JSON report).

  config 3: BER/BLER Monte-Carlo sweep, BG1 k=4096 rate 1/2, QPSK, Eb/N0 0-6 dB,
            error-count stopping (run_sweep, fast decoder) -> CSV + JSON
  config 4: 64-QAM APP vs max-log demapping, BG1 k=4096 n=12288 (rate 1/3, fillers,
            puncturing), batch 131072 -> throughput and BER/BLER at one Eb/N0
  config 5: decoder-only throughput, min-sum vs sum-product, 5-50 iterations,
            BG1/BG2 lifting sizes (specialised kernels where compiled, the runtime-Z
            kernel elsewhere)

  python tools/configs_report.py [--out profiles/r01/configs_report.json] [--quick]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2203_11854_b200 as lb  # noqa: E402


def config3(quick, outdir):
    pts = [0.0, 0.5, 1.0, 1.5, 2.0, 2.5, 3.0, 3.5, 4.0, 4.5, 5.0, 5.5, 6.0]
    res = {}
    for variant in ("min-sum", "sum-product"):
        cfg = lb.SimConfig.from_dict({
            "code": {"family": "ldpc5g", "k": 4096, "n": 8192,
                     "decoder": {"variant": variant, "mode": "fast", "num_iter": 20}},
            "modulation": {"kind": "qam", "bits_per_symbol": 2},
            "sweep": {"ebno_db": pts, "batch_size": 8192, "target_block_errors": 100,
                      "max_batches_per_point": 20 if quick else 300},
            "seed": 2024})
        t = time.perf_counter()
        r = lb.run_sweep(cfg, num_workers=8)  # waves of 8 batches, as the reference's worker pool
        torch.cuda.synchronize()
        el = time.perf_counter() - t
        csv = lb.format_csv(r)
        with open(os.path.join(outdir, f"sweep_c3_{variant}.csv"), "w") as f:
            f.write(csv)
        res[variant] = {"elapsed_s": el, "points": [
            {"ebno_db": p.ebno_db, "bits": p.bits, "bit_errors": p.bit_errors, "ber": p.ber,
             "blocks": p.blocks, "block_errors": p.block_errors, "bler": p.bler, "batches": p.batches,
             "stop_reason": p.stop_reason} for p in r.points],
            "decoded_bits": sum(p.bits for p in r.points),
            "throughput_gbit_s": sum(p.bits for p in r.points) / el / 1e9}
    return res


EB4 = 8.0  # 64-QAM rate 1/3 on the synthetic BG1 sits in its waterfall near 7-8 dB


def config4(quick):
    k, n, m = 4096, 12288, 6
    B = 16384 if quick else 131072
    out = {}
    for demapper in ("app", "maxlog"):
        cfg = lb.SimConfig.from_dict({
            "code": {"family": "ldpc5g", "k": k, "n": n,
                     "decoder": {"variant": "min-sum", "mode": "fast", "num_iter": 20, "early_stop": False}},
            "modulation": {"kind": "qam", "bits_per_symbol": m, "demapper": demapper},
            "sweep": {"ebno_db": [EB4], "batch_size": B}, "seed": 7})
        pipe = lb.Pipeline(cfg)
        counts = torch.zeros(2, dtype=torch.int64, device="cuda")
        pipe.run_batch_counts(EB4, B, lb.RngStream(7, 1), counts)
        torch.cuda.synchronize()
        counts.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        steps = 3
        for s in range(steps):
            pipe.run_batch_counts(EB4, B, lb.RngStream(7, 10 + s), counts)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        c = counts.cpu().tolist()
        out[demapper] = {"batch": B, "ebno_db": EB4, "ms_per_batch": ms, "gbit_s": B * k / ms / 1e6,
                         "ber": c[0] / (steps * B * k), "bler": c[1] / (steps * B),
                         "decoder_precision": pipe.precision, "fused_modem": pipe.fused_modem}
    return out


def config5(quick):
    """Decoder-only table: every lifting size in [32, 384],
    BG1 rate 1/2 and BG2 rate 1/3, 5-50 fixed iterations, min-sum and scaled
    min-sum on the fp16x2 decoder and sum-product (boxplus) on the fp16-message
    decoder (specialised instance where compiled, else the runtime-geometry
    kernel)."""
    iters = [5, 10, 20, 50]
    zs = [z for z in lb.ldpc.LIFTING_SIZES if 32 <= z <= 384] if not quick else [96, 384]
    rows = []
    for bg in (1, 2):
        kb = 22 if bg == 1 else 10
        for z in zs:
            k = kb * z
            n = 2 * k if bg == 1 else 3 * k
            code = lb.LdpcCode5G(k, n, base_graph=bg, z=z)
            B = max(256, min(65536, (1 << 26) // (68 * z)))
            B += B & 1
            torch.manual_seed(0)
            llr = (torch.randn(B, n, device="cuda") * 2.0 + 3.0).contiguous()  # all-zero codeword, ~4 dB
            edges = code.pcm.num_edges
            live = int(lb._lib.lib().ls_qc_live_rows(code.handle))
            for variant in ("min-sum", "scaled-min-sum", "sum-product"):
                prec = "fp32" if variant == "sum-product" else "fp16x2"
                spec = lb.ldpc.qc_has_kernel(code, prec, variant=variant)
                for it in iters:
                    lb.qc_decode(llr, code, it, variant, early_stop=False, want_hard=True, precision=prec)
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    lb.qc_decode(llr, code, it, variant, early_stop=False, want_hard=True, precision=prec)
                    e1.record()
                    torch.cuda.synchronize()
                    ms = e0.elapsed_time(e1)
                    kind = ("specialised " if spec else "runtime-geometry ") + (
                        "sum-product fp16" if variant == "sum-product" else "fp16x2")
                    rows.append({"bg": bg, "z": z, "k": k, "n": n, "variant": variant, "iters": it,
                                 "kernel": kind, "batch": B, "ms": ms, "info_gbit_s": B * k / ms / 1e6,
                                 "live_rows": live,
                                 "mother_graph_edge_updates_per_s": B * it * edges / (ms / 1e3)})
    return rows


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01", "configs_report.json"))
    p.add_argument("--quick", action="store_true")
    p.add_argument("--only", default="3,4,5")
    a = p.parse_args()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    rep = {}
    if os.path.exists(a.out):  # refresh only the configs asked for
        with open(a.out) as f:
            rep = json.load(f)
    rep["device"] = torch.cuda.get_device_name(0)
    if "3" in a.only:
        rep["config3_sweep"] = config3(a.quick, os.path.dirname(os.path.abspath(a.out)))
    if "4" in a.only:
        rep["config4_64qam"] = config4(a.quick)
    if "5" in a.only:
        rep["config5_decoder_only"] = config5(a.quick)
    with open(a.out, "w") as f:
        json.dump(rep, f, indent=1)
    print(json.dumps(rep)[:3000])


if __name__ == "__main__":
    main()
