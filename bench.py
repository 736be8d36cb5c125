"""Throughput benchmark of the coded-link hot path (BASELINE.json metric).

Workload (configs[1]): 5G LDPC BG1 k=8448 n=16896 (Z=384), 16-QAM over AWGN,
20 BP iterations, batch 65,536 codewords per GPU.  One step = one
Pipeline.run_batch of the chain binary_source -> ldpc5g_encode -> map_bits
-> awgn -> demap_app -> ldpc5g_decode -> count_errors on one batch of fresh
synthetic payload (new RngStream per step), all on the GPU.

  python bench.py [--gpus N --steps K --warmup W]            # B200 arm
  python bench.py --impl reference [...]                      # CPU reference arm

Under torchrun every rank runs its own batches (weak scaling, no data-path
collective); timing is CUDA events on the launching stream, max over ranks.
Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import concurrent.futures
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

K_INFO, N_TX, M_BITS = 8448, 16896, 4
# kernels of one headline step (ncu launch list, profiles/r02/launches_bench_r2h.csv):
# binary_source, encoder, mapper, 5 numpy-ziggurat kernels, noise apply, demapper, exact decoder
GPU_LAUNCHES_PER_STEP = 11
# DRAM bytes (read + write) per codeword of k_qc_exact<BG1,384,2>, from the
# ncu --set full capture of the bench's own 65,536-codeword decoder launch
# (profiles/r02/ncu_k_qc_exact_bench_r2h_summary.txt: 5.028 GB read + 18.2 MB
# written); the messages never leave the SM, DRAM sees the LLR input and the counts
EXACT_TRAFFIC_PER_CW = (5_027_535_000 + 18_208_768) / 65536
METRIC = "decoded info Gbit/s (LDPC BG1, 20 iters) at 1/2/4/8 B200 vs CPU ref; %roofline"


def _args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--batch", type=int, default=65536)
    p.add_argument("--variant", default="min-sum")
    p.add_argument("--iters", type=int, default=20)
    p.add_argument("--ebno", type=float, default=6.0)
    p.add_argument("--early-stop", action="store_true")
    p.add_argument("--seed", type=int, default=42)
    p.add_argument("--cpu-seconds", type=float, default=15.0)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-extra", action="store_true")
    return p.parse_args()


def _workload(a):
    return {"workload": f"chain BG1 k={K_INFO} n={N_TX} 16-QAM AWGN {a.ebno} dB, {a.variant}, "
                        f"{a.iters} iters {'early-stop' if a.early_stop else 'fixed'}",
            "code": "ldpc5g BG1 Z=384", "k": K_INFO, "n": N_TX, "modulation": "qam16",
            "batch_per_gpu": a.batch, "num_iter": a.iters, "variant": a.variant,
            "early_stop": bool(a.early_stop), "ebno_db": a.ebno,
            "l2": "inputs larger than L2 (fresh 4.4 GB LLR batch per step)"}


# ------------------------------------------------------------------ CPU (oracle port)
def cpu_chain_rate(a, seconds: float, threads: int):
    """Oracle port of Pipeline.run_batch on the host cores: `threads` workers
    each decoding batches of 4 codewords (the reference's [B,E] f64 working
    set limits per-worker batches) until `seconds`."""
    from oracle import linksim_oracle as O

    O.code(K_INFO, N_TX)  # build tables outside the timed region
    per = 4
    stop = time.perf_counter() + seconds
    done = []

    def worker(w):
        b = 0
        n = 0
        while time.perf_counter() < stop:
            O.run_batch(K_INFO, N_TX, M_BITS, a.ebno, per, a.seed, ((w + 1) << 32) | (b + 1), a.variant,
                        a.iters, "app", a.early_stop)
            b += 1
            n += per
        done.append(n)

    t0 = time.perf_counter()
    with concurrent.futures.ThreadPoolExecutor(threads) as ex:
        list(ex.map(worker, range(threads)))
    el = time.perf_counter() - t0
    cw = sum(done)
    return cw * K_INFO / el / 1e9, cw, el


def run_reference(a, rank):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    vals = []
    for _ in range(max(0, a.warmup) and 1):
        cpu_chain_rate(a, min(3.0, a.cpu_seconds), threads)
    total_cw = 0
    els = []
    for _ in range(a.steps):
        v, cw, el = cpu_chain_rate(a, a.cpu_seconds / max(1, a.steps) + 2.0, threads)
        vals.append(v)
        els.append(el)
        total_cw += cw
    v = sum(vals) / len(vals)
    # a reference step is one bounded wall-clock sample of the workload on all host threads
    ms = 1e3 * sum(els) / len(els)
    line = {"metric": METRIC, "value": v, "unit": "Gbit/s", "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64/f32 (reference precision pattern)", "data": "synthetic",
            "config": _workload(a), "impl": "reference",
            "cpu_baseline": dict({"value": v, "unit": "Gbit/s", "cores": threads, "kind": "port",
                                  "sample": f"{total_cw} codewords in batches of 4 per worker thread, "
                                            f"oracle port of run_batch (numpy + C BP)"}, **host_info()),
            "e2e": {"value": v, "unit": "Gbit/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ clocks
class Clocks:
    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(self.index)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            # a timed region shorter than the 100 ms sampling period still
            # gets one sample (taken right after it)
            t_end = time.perf_counter() + 1.0
            while not self.samples and time.perf_counter() < t_end:
                time.sleep(0.01)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max((float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for s in self.samples for j in range(4) if s[3 + j] == "Active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.samples)}


# ------------------------------------------------------------------ B200 arm
def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        return {}


def _roofline(B, bytes_cw, ms_per_launch, kernel, dec_ms, ms, traffic=None, note=None):
    peaks = _peaks()
    peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = B * bytes_cw / (ms_per_launch / 1e3) / 1e9
    r = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
         "traffic": traffic, "kernel": kernel, "bytes_per_codeword": bytes_cw, "codewords_per_launch": B,
         "kernel_ms_per_launch": ms_per_launch, "kernel_share_of_step": dec_ms / ms,
         "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)" if peaks else "fallback 6.65 TB/s"}
    if note:
        r["note"] = note
    return r


def _bytes_cw(iters):
    # VN-sweep model: I*4*N + 4*n + ceil(k/8) per codeword
    return iters * 4 * 68 * 384 + 4 * N_TX + (K_INFO + 7) // 8


def run_b200(a, rank, world, local_rank):
    import torch

    import paper_2203_11854_b200 as lb
    from paper_2203_11854_b200 import _lib as L

    # LS_BENCH_BACKEND=gloo only exists to exercise the multi-rank code path
    # on a single-GPU box (ranks then share the device; timings meaningless)
    backend = os.environ.get("LS_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local_rank %= torch.cuda.device_count()
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    # the headline chain is the reference's own arithmetic end to end: numpy-exact
    # payload and noise streams, f64 demapper cast to f32, and the on-chip exact
    # BP decoder (bit-identical to ldpc.py:86-172) over the whole mother graph
    cfg = lb.SimConfig.from_dict({
        "code": {"family": "ldpc5g", "k": K_INFO, "n": N_TX,
                 "decoder": {"variant": a.variant, "num_iter": a.iters, "mode": "exact"}},
        "modulation": {"kind": "qam", "bits_per_symbol": M_BITS},
        "sweep": {"ebno_db": [a.ebno], "batch_size": a.batch}, "seed": a.seed})
    pipe = lb.Pipeline(cfg)
    assert pipe.qc_exact, "the on-chip exact decoder instance for config 2 is missing"
    B = a.batch
    counts = L.zeros((2,), "int64")
    stream = torch.cuda.current_stream()

    def rng(step):
        return lb.RngStream(a.seed, ((rank + 1) << 40) | (step + 1))

    dec_events = []

    def step(i, timed):
        payload, llr = pipe._llr(a.ebno, B, rng(i))
        if timed:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        lb.qc_decode(llr, pipe.ldpc, a.iters, a.variant, 0.75, early_stop=a.early_stop, ref_bits=payload,
                     want_hard=False, counts=counts, precision="exact")
        if timed:
            e1.record(stream)
            dec_events.append((e0, e1))

    for i in range(a.warmup):
        step(10_000 + i, False)
    torch.cuda.synchronize()
    counts.zero_()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local_rank) as clk:
        t0.record(stream)
        for i in range(a.steps):
            step(i, True)
        t1.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms = t0.elapsed_time(t1)
    dec_ms = sum(e0.elapsed_time(e1) for e0, e1 in dec_events)
    tm = torch.tensor([ms, dec_ms], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    ms, dec_ms = float(tm[0]), float(tm[1])
    errs = counts.cpu().tolist()
    value = world * B * K_INFO * a.steps / (ms / 1e3) / 1e9
    line = {"metric": METRIC, "value": value, "unit": "Gbit/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32 posteriors / f64 messages (reference arithmetic, bit-exact)",
            "data": "synthetic (random payload per step)",
            "config": dict(_workload(a), decoder="exact (on-chip, bit-identical to the reference)",
                           noise="numpy-exact ziggurat replica", demapper="app f64 -> f32"),
            "gpu_launches": GPU_LAUNCHES_PER_STEP * a.steps,
            "roofline": _roofline(B, _bytes_cw(a.iters), dec_ms / a.steps, "k_qc_exact<BG1,384,2>", dec_ms, ms,
                                  traffic=EXACT_TRAFFIC_PER_CW * B,
                                  note="messages stay on chip (f64 min1 + argmin/sign words in shared memory, "
                                       "min2 and channel in an L2 slice per SM); the kernel is bound by the "
                                       "ALU issue pipe, not HBM (ncu in profiles/r02)"),
            "issue_roofline": {"note": "from the ncu --set full capture of this decoder launch at B=65,536 "
                                       "(profiles/r02/ncu_k_qc_exact_bench_r2h_summary.txt)",
                               "warp_instructions_per_launch": 180_086_345_950, "ipc": 2.67, "ipc_peak": 4.0,
                               "issue_frac": 2.67 / 4.0, "alu_pipe_frac": 0.691,
                               "dram_bytes_per_launch": 5_045_743_768},
            "clocks": clk.summary(),
            "errors_in_timed_region": {"bit_errors": errs[0], "block_errors": errs[1],
                                       "blocks": world * B * a.steps}}
    if not a.no_e2e:
        line["e2e"] = e2e_decode(a, pipe, rank, world, dist)
        line["e2e_run_batch"] = e2e_chain(a, pipe, rank, world, dist)
    if not a.no_extra:
        line["exact_early_stop"] = exact_early_stop_rate(a, pipe, rank, world, dist)
        line["fast_fp16x2_min_sum"] = fast_rate(a, rank, world, dist, "fp16x2", prune=True)
        line["fast_fp32_full_graph"] = fast_rate(a, rank, world, dist, "fp32-full", prune=False)
        line["sum_product_fast"] = sum_product_rate(a, rank, world, dist)
        if rank == 0:
            line["sum_product_f32"] = sum_product_f32_rate(a)
        line["config3_sweep"] = config3_sweep(a, rank, world, dist)
        line["config4_demappers"] = config4_demappers(a, rank, world, dist)
        if rank == 0:
            line["config5_decoder_only"] = config5_decoder_only(a)
    if rank == 0 and world == 1 and not a.no_cpu:
        v, cw, el = cpu_chain_rate(a, a.cpu_seconds, os.cpu_count() or 1)
        line["cpu_baseline"] = dict({"value": v, "unit": "Gbit/s", "cores": os.cpu_count() or 1, "kind": "port",
                                     "sample": f"{cw} codewords ({el:.1f} s), oracle port of run_batch, "
                                               f"batches of 4 per worker thread"}, **host_info())
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def host_info():
    """Host facts BASELINE.md section 3 asks for beside a CPU number."""
    info = {"threads_used": os.cpu_count() or 1,
            "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS", "unset (default)")}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                info["cpu_model"] = line.split(":", 1)[1].strip()
            if line.startswith("Socket(s):") or line.startswith("Core(s) per socket:"):
                info[line.split(":")[0].strip().lower().replace(" ", "_")] = line.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    try:
        import numpy as np
        import scipy

        info["numpy"] = np.__version__
        info["scipy"] = scipy.__version__
        try:
            cfg = np.show_config(mode="dicts")
            blas = cfg.get("Build Dependencies", {}).get("blas", {})
            info["blas"] = f"{blas.get('name', '?')} {blas.get('version', '')}".strip()
        except Exception:  # pragma: no cover - numpy without the dict mode
            pass
    except ImportError:  # pragma: no cover
        pass
    info["note"] = ("oracle port (numpy + the C restatement of bp_decode), ~50x faster than the numpy "
                    "reference itself (BASELINE.md section 4), so the GPU/CPU ratio is conservative")
    return info


def _timed_steps(fn, steps, dist, reset=None):
    import torch

    fn(-1)
    torch.cuda.synchronize()
    if reset:
        reset()
    if dist:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(torch.cuda.current_device()) as clk:
        e0.record()
        for i in range(steps):
            fn(i)
        e1.record()
        torch.cuda.synchronize()
    tm = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    return float(tm[0]), clk.summary()


def exact_early_stop_rate(a, pipe, rank, world, dist, steps=3):
    """The exact chain with the reference's syndrome early stop (ldpc.py:155-167;
    converged codewords leave the persistent decoder at once)."""
    import torch

    import paper_2203_11854_b200 as lb
    from paper_2203_11854_b200 import _lib as L

    B = a.batch
    counts = L.zeros((2,), "int64")
    iters = []

    def one(i):
        payload, llr = pipe._llr(a.ebno, B, lb.RngStream(a.seed, ((rank + 1) << 40) | (900 + i)))
        r = lb.qc_decode(llr, pipe.ldpc, a.iters, a.variant, 0.75, early_stop=True, ref_bits=payload,
                         want_hard=False, want_iters=True, counts=counts, precision="exact")
        iters.append(r["iters"])

    ms, clk = _timed_steps(one, steps, dist, reset=counts.zero_)
    mean_it = float(torch.cat(iters[1:]).float().mean())
    return {"value": world * B * K_INFO * steps / (ms / 1e3) / 1e9, "unit": "Gbit/s",
            "mean_iterations": mean_it, "ms_per_step": ms / steps, "clocks": clk,
            "note": "exact chain, early stop as the reference (per-codeword syndrome after each iteration)"}


def _fast_pipe(a, variant):
    import paper_2203_11854_b200 as lb

    cfg = lb.SimConfig.from_dict({
        "code": {"family": "ldpc5g", "k": K_INFO, "n": N_TX,
                 "decoder": {"variant": variant, "num_iter": a.iters, "mode": "fast", "early_stop": False}},
        "modulation": {"kind": "qam", "bits_per_symbol": M_BITS},
        "sweep": {"ebno_db": [a.ebno], "batch_size": a.batch}, "seed": a.seed})
    return lb.Pipeline(cfg)


def fast_rate(a, rank, world, dist, precision, prune, steps=3):
    """Statistically-equivalent fast chain (fused Philox modem + on-chip
    decoder), labelled: not the reference arithmetic."""
    import torch

    import paper_2203_11854_b200 as lb
    from paper_2203_11854_b200 import _lib as L

    pipe = _fast_pipe(a, a.variant)
    B = a.batch
    counts = L.zeros((2,), "int64")
    dec = []

    def one(i):
        payload, llr = pipe._llr(a.ebno, B, lb.RngStream(a.seed, ((rank + 1) << 40) | (700 + i)))
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d0.record()
        lb.qc_decode(llr, pipe.ldpc, a.iters, a.variant, 0.75, early_stop=False, ref_bits=payload,
                     want_hard=False, counts=counts, precision=precision, prune=prune)
        d1.record()
        dec.append((d0, d1))

    ms, clk = _timed_steps(one, steps, dist, reset=counts.zero_)
    dms = sum(d0.elapsed_time(d1) for d0, d1 in dec[1:]) / steps
    c = counts.cpu().tolist()
    return {"value": world * B * K_INFO * steps / (ms / 1e3) / 1e9, "unit": "Gbit/s", "ms_per_step": ms / steps,
            "decoder_ms_per_launch": dms, "decoder_gbit_s": B * K_INFO / (dms / 1e3) / 1e9,
            "dtype": "f16x2" if precision == "fp16x2" else "f32",
            "kernel": {"fp16x2": "k_qc_fast_h2w", "fp32-full": "k_qc_exact<BG1,384,2,float>"}.get(precision, precision),
            "rows": "24 live rows (dead extension rows pruned)" if prune else "all 46 rows",
            "roofline_frac": B * _bytes_cw(a.iters) / (dms / 1e3) / 1e9 / float(_peaks().get("hbm_gbs", 6650.0)),
            # DRAM bytes per launch at B=65,536 from ncu --set full (profiles/r02/ncu_*_bench_summary.txt)
            "traffic_per_launch_at_65536": {"fp16x2": 4_992_890_000 + 5_429_504,
                                            "fp32-full": 5_013_454_000 + 9_787_904}.get(precision),
            "bit_errors": c[0], "block_errors": c[1], "clocks": clk,
            "note": "fast mode: Philox noise, f32 modem, narrower message arithmetic; statistically "
                    "equivalent to the reference, not bit-exact"}


def sum_product_rate(a, rank, world, dist, steps=2):
    """The reference's default BP variant (sum-product, ldpc.py:139-143), fast
    mode, fixed iterations: fp16 per-edge messages on chip, fp32 math."""
    import torch

    import paper_2203_11854_b200 as lb
    from paper_2203_11854_b200 import _lib as L

    pipe = _fast_pipe(a, "sum-product")
    B = a.batch
    counts = L.zeros((2,), "int64")
    dec = []

    def one(i):
        payload, llr = pipe._llr(a.ebno, B, lb.RngStream(a.seed, ((rank + 1) << 40) | (600 + i)))
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d0.record()
        lb.qc_decode(llr, pipe.ldpc, a.iters, "sum-product", early_stop=False, ref_bits=payload, want_hard=False,
                     counts=counts)
        d1.record()
        dec.append((d0, d1))

    ms, clk = _timed_steps(one, steps, dist, reset=counts.zero_)
    dms = sum(d0.elapsed_time(d1) for d0, d1 in dec[1:]) / steps
    c = counts.cpu().tolist()
    return {"value": world * B * K_INFO * steps / (ms / 1e3) / 1e9, "unit": "Gbit/s", "ms_per_step": ms / steps,
            "decoder_ms_per_launch": dms, "bit_errors": c[0], "block_errors": c[1], "clocks": clk,
            "note": "sum-product, fixed iterations, k_qc_sp (fp16 messages in shared memory, fp32 base-2 phi, "
                    "product-domain check update); fast mode, statistically equivalent"}


def config3_sweep(a, rank, world, dist):
    """BASELINE config 3: error-count-stopped Eb/N0 sweep, BG1 k=4096 r=1/2
    QPSK, exact decoder (the reference's arithmetic), waves of batches sharded
    over the ranks (sweep.py:411-476).  Bounded: 4 batches of 8,192 per point."""
    import torch

    import paper_2203_11854_b200 as lb

    cfg = lb.SimConfig.from_dict({
        "code": {"family": "ldpc5g", "k": 4096, "n": 8192, "decoder": {"variant": "min-sum", "num_iter": 20}},
        "modulation": {"kind": "qam", "bits_per_symbol": 2},
        "sweep": {"ebno_db": [0.0, 1.0, 2.0, 3.0, 4.0, 5.0, 6.0], "batch_size": 8192,
                  "target_block_errors": 100, "max_batches_per_point": 4}, "seed": 2024})
    lb.run_sweep(lb.SimConfig.from_dict({  # warm-up (handles, workspaces)
        "code": cfg.code, "modulation": cfg.modulation,
        "sweep": {"ebno_db": [3.0], "batch_size": 8192, "max_batches_per_point": 1}}), num_workers=1)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t = time.perf_counter()
    # one batch per rank per stopping check (the reference's default
    # num_workers=1, sweep.py:411): a wider wave only computes batches the
    # prefix-truncation rule then discards at the high-BLER points
    res = lb.run_sweep(cfg, num_workers=world)
    torch.cuda.synchronize()
    el = _wall_max(dist, time.perf_counter() - t)
    bits = sum(p.bits for p in res.points)
    return {"value": bits / el / 1e9, "unit": "Gbit/s", "decoded_bits": bits, "elapsed_s": el,
            "points": [[p.ebno_db, p.blocks, p.block_errors, p.bit_errors, p.stop_reason] for p in res.points],
            "note": "run_sweep, exact mode (numpy-exact noise, on-chip exact decoder, Z=192: two codewords per "
                    "CTA in lockstep), waves of one batch per rank; statistics identical for any rank or worker "
                    "count; wall clock incl. host orchestration; decoded_bits counts the kept batches only"}


def config4_demappers(a, rank, world, dist, B=131072):
    """BASELINE config 4: 64-QAM APP vs max-log, BG1 k=4096 n=12288 (r=1/3,
    fillers, puncturing), batch 131,072, exact chain."""
    import paper_2203_11854_b200 as lb
    from paper_2203_11854_b200 import _lib as L

    out = {}
    for demapper in ("app", "maxlog"):
        pipe = lb.Pipeline(lb.SimConfig.from_dict({
            "code": {"family": "ldpc5g", "k": 4096, "n": 12288, "decoder": {"variant": "min-sum", "num_iter": 20}},
            "modulation": {"kind": "qam", "bits_per_symbol": 6, "demapper": demapper},
            "sweep": {"ebno_db": [7.5], "batch_size": B}, "seed": 7}))
        counts = L.zeros((2,), "int64")

        def one(i):
            pipe.run_batch_counts(7.5, B, lb.RngStream(7, ((rank + 1) << 40) | (20 + i)), counts)

        ms, clk = _timed_steps(one, 2, dist, reset=counts.zero_)
        c = counts.cpu().tolist()
        out[demapper] = {"value": world * B * 4096 * 2 / (ms / 1e3) / 1e9, "unit": "Gbit/s", "ms_per_step": ms / 2,
                         "bit_errors": c[0], "block_errors": c[1], "blocks": 2 * B, "clocks": clk}
    out["note"] = "exact chain at 7.5 dB (numpy-exact noise, f64 demapper, on-chip exact decoder, early stop on)"
    return out


def config5_decoder_only(a):
    """BASELINE config 5 (subset): decoder-only throughput, min-sum vs
    sum-product (boxplus), 5/20/50 iterations, BG1 and BG2 at Z = 64..384."""
    import torch

    import paper_2203_11854_b200 as lb

    rows = []
    for bg, z in ((1, 64), (1, 192), (1, 384), (2, 64), (2, 384)):
        kb = 22 if bg == 1 else 10
        k = kb * z
        n = 2 * k if bg == 1 else 3 * k
        code = lb.LdpcCode5G(k, n, base_graph=bg, z=z)
        B = max(1024, (1 << 27) // k)
        cfgd = {"code": {"family": "ldpc5g", "k": k, "n": n, "decoder": {"mode": "fast"}},
                "modulation": {"kind": "qam", "bits_per_symbol": 2}, "sweep": {"ebno_db": [4.0], "batch_size": B}}
        pipe = lb.Pipeline(lb.SimConfig.from_dict(cfgd))
        pipe.ldpc = code
        payload, llr = pipe._llr(4.0 if bg == 1 else 5.0, B, lb.RngStream(5, z))
        kinds = [("min-sum", "fp16x2"), ("sum-product", "fp32")]
        if lb.ldpc.qc_has_kernel(code, precision="exact"):
            kinds += [("min-sum", "exact"), ("min-sum", "fp32-full")]
        for variant, prec in kinds:
            for it in (5, 20, 50):
                def run():
                    return lb.qc_decode(llr, code, it, variant, 0.75, early_stop=False, want_hard=False,
                                        ref_bits=payload, precision=prec)
                try:
                    run()
                except ValueError as e:  # no instance for this geometry
                    rows.append({"bg": bg, "z": z, "variant": variant, "precision": prec, "iters": it,
                                 "skipped": str(e)})
                    continue
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                run()
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1)
                rows.append({"bg": bg, "z": z, "k": k, "n": n, "variant": variant, "precision": prec, "iters": it,
                             "batch": B, "ms": ms, "gbit_s": B * k / (ms / 1e3) / 1e9})
    return {"rows": rows, "note": "decoder only on device-resident LLRs (fast modem), fixed iterations; BG2 at "
                                  "Z >= 32 is the harness-lifted graph (LdpcCode5G(k, n, base_graph=2, z=Z))"}


def _sp_rates(a, k, n, m, ebno, B):
    import torch

    import paper_2203_11854_b200 as lb

    pipe = lb.Pipeline(lb.SimConfig.from_dict({
        "code": {"family": "ldpc5g", "k": k, "n": n, "decoder": {"mode": "fast"}},
        "modulation": {"kind": "qam", "bits_per_symbol": m}, "sweep": {"ebno_db": [ebno], "batch_size": B}}))
    payload, llr = pipe._llr(ebno, B, lb.RngStream(a.seed, 31))
    out = {}
    for prec in ("fp32-full", "fp32"):
        def run():
            return lb.qc_decode(llr, pipe.ldpc, a.iters, "sum-product", early_stop=False, ref_bits=payload,
                                want_hard=False, precision=prec)
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        out["f32_messages" if prec == "fp32-full" else "fp16_messages"] = {
            "ms": ms, "gbit_s": B * k / (ms / 1e3) / 1e9}
    return out


def sum_product_f32_rate(a, B=32768):
    """The f32-message sum-product option (k_qc_sp32, within 1e-4 of exact
    sum-product on converged codewords) next to the fp16-message kernel, on
    config 3 (BG1 k=4096 r=1/2, Z=192: f32 messages in shared memory) and
    config 2 (Z=384: f32 messages in an L2 slice per CTA)."""
    out = _sp_rates(a, 4096, 8192, 2, 2.0, B)
    out["config2"] = _sp_rates(a, K_INFO, N_TX, M_BITS, 4.8, B // 2)
    out["note"] = ("decoder only, 20 fixed iterations, config 3 at 2.0 dB (config2: 4.8 dB); f32 messages: "
                   "k_qc_sp32 (3 MUFU per edge, division-free product domain with prefix/suffix products; "
                   "config 2: messages in L2); fp16 messages: k_qc_sp (4 MUFU, product domain)")
    return out


def _wall_max(dist, secs):
    import torch

    if not dist:
        return secs
    t = torch.tensor([secs], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t[0])


def e2e_chain(a, pipe, rank, world, dist, steps=3):
    """The public API call a user makes (Pipeline.run_batch, sweep.py:347):
    host numpy (payload, decoded) out every step; exact chain."""
    import torch

    import paper_2203_11854_b200 as lb

    B = a.batch
    p, d = pipe.run_batch(a.ebno, B, lb.RngStream(a.seed, 98))
    p, d = pipe.run_batch(a.ebno, B, lb.RngStream(a.seed, 99))
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t = time.perf_counter()
    for i in range(steps):
        p, d = pipe.run_batch(a.ebno, B, lb.RngStream(a.seed, ((rank + 1) << 40) | (500 + i)))
    torch.cuda.synchronize()
    el = _wall_max(dist, time.perf_counter() - t)
    return {"value": world * B * K_INFO * steps / el / 1e9, "unit": "Gbit/s", "h2d_bytes_per_step": 0,
            "d2h_bytes_per_step": 2 * B * K_INFO,
            "api": "Pipeline.run_batch -> numpy (payload, decoded); inputs are the RngStream keys; the "
                   "reference's Pipeline semantics, i.e. the decoder's early stop is on (sweep.py:335-336)"}


def e2e_decode(a, pipe, rank, world, dist, steps=3):
    """The drop-in decoder with HOST buffers: pinned f32 LLRs in, decoded bits
    out (ldpc5g_decode(llr, code), exact mode, ldpc.py:354-365): the H2D copy
    of each step's LLRs and the D2H copy of its bits are inside the timed region."""
    import torch

    import paper_2203_11854_b200 as lb

    B = a.batch
    _, llr = pipe._llr(a.ebno, B, lb.RngStream(a.seed, 77))
    host = torch.empty(llr.shape, dtype=torch.float32, pin_memory=True)
    host.copy_(llr)
    del llr
    for _ in range(2):  # steady state of the pinned-host caching allocator
        dec = lb.ldpc5g_decode(host, pipe.ldpc, a.iters, a.variant, mode="exact", early_stop=a.early_stop)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t = time.perf_counter()
    for _ in range(steps):
        dec = lb.ldpc5g_decode(host, pipe.ldpc, a.iters, a.variant, mode="exact", early_stop=a.early_stop)
        assert dec.device.type == "cpu" and dec.shape == (B, K_INFO)  # decoded bits are on the host
    torch.cuda.synchronize()
    el = _wall_max(dist, time.perf_counter() - t)
    return {"value": world * B * K_INFO * steps / el / 1e9, "unit": "Gbit/s",
            "h2d_bytes_per_step": 4 * B * N_TX, "d2h_bytes_per_step": B * K_INFO,
            "api": "ldpc5g_decode(pinned host f32 LLRs, mode='exact') -> host bits (copies overlap the decoder "
                   "in 2,048-row chunks)"}


def main():
    a = _args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        run_reference(a, rank)
        return
    run_b200(a, rank, world, local_rank)


if __name__ == "__main__":
    main()
