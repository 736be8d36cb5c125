"""Monte-Carlo BER/BLER sweep on B200 (mirror of linksim.sweep, sweep.py:1-520).

Scope: the AWGN + 5G-LDPC (and uncoded "none") pipeline of the hot path.
Config validation, CSV format, RNG keying (seed, snr_idx, batch_idx) and the
deterministic stopping rule are the reference's, so a sweep gives the same
statistics for any number of GPUs, as the reference does for any number of
worker threads (sweep.py:425-476; test_acceptance.py:329-337).

Multi-GPU: one process per GPU (torch.distributed, NCCL).  Batch indices of
each wave are dealt round-robin to ranks; the only collective is an
all_gather of the per-batch (bit_errors, block_errors) int64 pairs, after
which every rank applies the identical prefix-truncation rule.
"""
from __future__ import annotations

import csv
import io
import time
from dataclasses import dataclass, field

from . import _lib as L
from .channel import awgn
from .core import RngStream, binary_source, ebnodb2no
from .ldpc import BP_VARIANTS, LdpcCode5G, ldpc5g_decode, ldpc5g_encode, qc_decode, qc_has_kernel
from .mapping import Constellation, demap_app, demap_maxlog, map_bits, modem_qam

CSV_COLUMNS = ("ebno_db", "bits", "bit_errors", "ber", "blocks", "block_errors", "bler", "batches",
               "stop_reason", "elapsed_s")
DEFAULT_TARGET_BLOCK_ERRORS = 100
DEFAULT_MAX_BATCHES = 1000


class ConfigError(ValueError):
    """Invalid simulation config; names the offending field (sweep.py:37-42)."""

    def __init__(self, fieldname: str, message: str):
        super().__init__(f"{fieldname}: {message}")
        self.field = fieldname


def _req(d: dict, dotted: str):
    key = dotted.split(".")[-1]
    if key not in d:
        raise ConfigError(dotted, "missing required field")
    return d[key]


@dataclass
class SimConfig:
    code: dict
    modulation: dict
    channel: dict
    ofdm: dict
    mimo: dict
    snr_points: list
    batch_size: int
    target_block_errors: int
    max_batches_per_point: int
    seed: int
    precision: str

    @classmethod
    def from_dict(cls, raw: dict) -> "SimConfig":
        """Validate like sweep.py:68-136; branches outside the hot path
        (polar/conv codes, flat/TDL channels, OFDM, MIMO) are rejected with a
        ConfigError naming the field."""
        if not isinstance(raw, dict):
            raise ConfigError("<root>", "config must be a JSON object")
        code = dict(raw.get("code", {"family": "none", "k": 100}))
        family = _req(code, "code.family")
        if family not in ("none", "ldpc5g", "polar5g", "conv"):
            raise ConfigError("code.family", f"unknown family {family!r}")
        if family in ("polar5g", "conv"):
            raise ConfigError("code.family", f"family {family!r} is not on the B200 path")
        k = _req(code, "code.k")
        if not isinstance(k, int) or k < 1:
            raise ConfigError("code.k", "must be a positive integer")
        if family == "ldpc5g":
            n = _req(code, "code.n")
            if not isinstance(n, int) or n <= k:
                raise ConfigError("code.n", "must be an integer > k")
        modulation = dict(raw.get("modulation", {"kind": "qam", "bits_per_symbol": 2}))
        kind = modulation.get("kind", "qam")
        if kind not in ("qam", "psk"):
            raise ConfigError("modulation.kind", f"unknown kind {kind!r}")
        m = modulation.get("bits_per_symbol")
        if not isinstance(m, int) or m < 1:
            raise ConfigError("modulation.bits_per_symbol", "must be a positive integer")
        if kind == "qam" and m % 2:
            raise ConfigError("modulation.bits_per_symbol", "qam needs an even value")
        chan = dict(raw.get("channel", {"kind": "awgn"}))
        ck = chan.get("kind", "awgn")
        if ck not in ("awgn", "flat", "tdl"):
            raise ConfigError("channel.kind", f"unknown kind {ck!r}")
        if ck != "awgn":
            raise ConfigError("channel.kind", f"channel {ck!r} is not on the B200 path")
        ofdm_cfg = dict(raw.get("ofdm", {"enabled": False}))
        mimo_cfg = dict(raw.get("mimo", {"enabled": False}))
        if ofdm_cfg.get("enabled"):
            raise ConfigError("ofdm.enabled", "OFDM is not on the B200 path")
        if mimo_cfg.get("enabled"):
            raise ConfigError("mimo.enabled", "MIMO is not on the B200 path")
        sweep = dict(_req(raw, "sweep"))
        points = _req(sweep, "sweep.ebno_db")
        if (not isinstance(points, list) or not points
                or any(isinstance(p, bool) or not isinstance(p, (int, float)) for p in points)):
            raise ConfigError("sweep.ebno_db", "must be a non-empty list of numbers")
        if any(b <= a for a, b in zip(points, points[1:])):
            raise ConfigError("sweep.ebno_db", "must be strictly increasing")
        batch_size = sweep.get("batch_size", 256)
        if not isinstance(batch_size, int) or batch_size < 1:
            raise ConfigError("sweep.batch_size", "must be a positive integer")
        precision = raw.get("precision", "single")
        if precision not in ("single", "double"):
            raise ConfigError("precision", "must be 'single' or 'double'")
        cfg = cls(code=code, modulation=modulation, channel=chan, ofdm=ofdm_cfg, mimo=mimo_cfg,
                  snr_points=[float(p) for p in points], batch_size=batch_size,
                  target_block_errors=sweep.get("target_block_errors", DEFAULT_TARGET_BLOCK_ERRORS),
                  max_batches_per_point=sweep.get("max_batches_per_point", DEFAULT_MAX_BATCHES),
                  seed=raw.get("seed", 0), precision=precision)
        build_pipeline(cfg)
        return cfg


@dataclass
class SnrPointResult:
    ebno_db: float
    bits: int
    bit_errors: int
    blocks: int
    block_errors: int
    batches: int
    stop_reason: str
    elapsed_s: float

    @property
    def ber(self) -> float:
        return self.bit_errors / self.bits if self.bits else 0.0

    @property
    def bler(self) -> float:
        return self.block_errors / self.blocks if self.blocks else 0.0


@dataclass
class SweepResult:
    config: SimConfig
    points: list = field(default_factory=list)


class Pipeline:
    """AWGN coded-link chain for one config (sweep.py:165-364) on the GPU."""

    def __init__(self, cfg: SimConfig):
        self.cfg = cfg
        mod = cfg.modulation
        self.constellation = Constellation(mod.get("kind", "qam"), mod["bits_per_symbol"])
        self.m = mod["bits_per_symbol"]
        demapper = mod.get("demapper", "app")
        if demapper not in ("app", "maxlog"):
            raise ConfigError("modulation.demapper", f"unknown demapper {demapper!r}")
        self.demapper = demapper
        self.demap = demap_app if demapper == "app" else demap_maxlog
        code = cfg.code
        self.family = code["family"]
        dec = dict(code.get("decoder", {}))
        if self.family == "none":
            self.payload_bits = self.coded_bits = code["k"]
            self.coderate = 1.0
        else:
            self.ldpc = LdpcCode5G(code["k"], code["n"])
            variant = dec.get("variant", "sum-product")
            if variant not in BP_VARIANTS:
                raise ConfigError("code.decoder.variant", f"unknown variant {variant!r}")
            self.bp_variant = variant
            self.bp_iter = dec.get("num_iter", 20)
            self.decoder_mode = dec.get("mode", "exact")
            if self.decoder_mode not in ("exact", "fast"):
                raise ConfigError("code.decoder.mode", f"unknown mode {self.decoder_mode!r}")
            # The reference's Pipeline decodes with ldpc5g_decode's defaults
            # (scale 0.75, early stop on) whatever the config says
            # (sweep.py:335-336).  Exact mode keeps that drop-in behaviour;
            # decoder.scale / decoder.early_stop are B200 fast-mode options.
            self.bp_scale, self.bp_early_stop = 0.75, True
            if self.decoder_mode == "fast":
                self.bp_scale = dec.get("scale", 0.75)
                self.bp_early_stop = dec.get("early_stop", True)
            elif dec.get("scale", 0.75) != 0.75 or dec.get("early_stop", True) is not True:
                import warnings

                warnings.warn("code.decoder.scale / early_stop are ignored in exact mode, as by the "
                              "reference's Pipeline (sweep.py:335-336); set decoder.mode 'fast' to use them",
                              stacklevel=2)
            self.decoder_precision = dec.get("precision", "auto")
            if self.decoder_precision not in ("auto", "fp32", "fp16x2", "fp32-full"):
                raise ConfigError("code.decoder.precision",
                                  f"unknown precision {self.decoder_precision!r}")
            if cfg.precision == "double" and self.decoder_mode != "exact":
                raise ConfigError("precision", "'double' runs the exact f64 chain; decoder.mode 'fast' "
                                               "computes in f32 / fp16")
            self.payload_bits = code["k"]
            self.coded_bits = code["n"]
            self.coderate = code["k"] / code["n"]
        if self.coded_bits % self.m:
            raise ConfigError("modulation.bits_per_symbol",
                              f"coded block of {self.coded_bits} bits is not divisible by "
                              f"{self.m} bits/symbol")
        self.num_symbols = self.coded_bits // self.m
        _ = self.noise  # validates channel.noise

    # -- per-batch simulation (device resident) ------------------------------
    @property
    def noise(self) -> str:
        """'numpy' (the reference's exact draws) unless the fast decoder is
        selected; `channel.noise` overrides."""
        default = "philox" if (self.family != "none" and self.decoder_mode == "fast") else "numpy"
        kind = self.cfg.channel.get("noise", default)
        if kind not in ("numpy", "philox"):
            raise ConfigError("channel.noise", f"unknown noise generator {kind!r}")
        return kind

    @property
    def fused_modem(self) -> bool:
        """Fast chain: one fused map+AWGN+demap pass for Gray QAM."""
        return (self.family != "none" and self.decoder_mode == "fast" and self.noise == "philox"
                and self.cfg.precision == "single" and self.constellation.qam_axes() is not None)

    def _llr(self, ebno_db: float, batch_size: int, rng: RngStream, lo: int = 0):
        """Payload and f32 LLRs of rows [lo, lo + batch_size) of a batch: the
        random streams are addressed by row, so a batch computed in chunks is
        identical to one computed at once (lo must be a multiple of 32)."""
        no = ebnodb2no(ebno_db, self.m, self.coderate)
        payload = binary_source([batch_size, self.payload_bits], rng.child(0), device=True,
                                offset=lo * self.payload_bits)
        coded = payload if self.family == "none" else ldpc5g_encode(payload, self.ldpc, device=True)
        sym0 = lo * self.num_symbols
        if self.fused_modem:
            llr = modem_qam(coded, self.constellation, no, rng.child(2), self.demapper, offset=sym0)
            return payload, llr
        double = self.cfg.precision == "double"  # complex128 symbols, f64 LLRs (sweep.py:170, 352, 362)
        x = map_bits(coded, self.constellation, device=True, dtype="complex128" if double else "complex64")
        y = awgn(x, no, rng.child(2), device=True, offset=sym0, noise=self.noise)
        llr = self.demap(y, no, self.constellation, out_dtype="float64" if double else "float32", device=True)
        return payload, llr

    @property
    def qc_exact(self) -> bool:
        """Exact mode served by the on-chip QC decoder (min-sum variants on
        f32 LLRs; precision 'double' decodes f64 LLRs on the CSR engine)."""
        if self.family == "none" or self.decoder_mode != "exact" or self.cfg.precision == "double":
            return False
        if getattr(self, "_qc_exact", None) is None:
            self._qc_exact = qc_has_kernel(self.ldpc, precision="exact", variant=self.bp_variant)
        return self._qc_exact

    @property
    def precision(self) -> str:
        if self.decoder_precision != "auto":
            return self.decoder_precision
        return "fp16x2"

    def run_batch_device(self, ebno_db: float, batch_size: int, rng: RngStream, lo: int = 0):
        """(payload, decoded) as CUDA tensors (rows [lo, lo + batch_size))."""
        payload, llr = self._llr(ebno_db, batch_size, rng, lo)
        if self.family == "none":
            return payload, (llr > 0).to(L.torch().uint8)
        if self.decoder_mode == "fast":
            dec = qc_decode(llr, self.ldpc, self.bp_iter, self.bp_variant, self.bp_scale,
                            early_stop=self.bp_early_stop, precision=self.precision)["hard"]
        else:
            dec = ldpc5g_decode(llr, self.ldpc, self.bp_iter, self.bp_variant, self.bp_scale,
                                mode="exact", early_stop=self.bp_early_stop, device=True)
        return payload, dec

    def run_batch(self, ebno_db: float, batch_size: int, rng: RngStream, chunk: int = 4096):
        """Simulate one batch; returns (payload, decoded) numpy bit arrays (sweep.py:347-364).

        The batch runs in row chunks; each chunk's results are copied to
        pinned host memory on a side stream while the next chunk computes.
        """
        torch = L.torch()
        if batch_size <= chunk or self.noise == "numpy":  # the numpy stream is drawn per batch
            p, d = self.run_batch_device(ebno_db, batch_size, rng)
            # pinned outputs from torch's caching host allocator: one fast D2H
            # each, and the numpy arrays keep their buffers alive
            ph = torch.empty(tuple(p.shape), dtype=p.dtype, pin_memory=True)
            dh = torch.empty(tuple(d.shape), dtype=d.dtype, pin_memory=True)
            ph.copy_(p, non_blocking=True)
            dh.copy_(d, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            return ph.numpy(), dh.numpy()
        chunk = max(32, (chunk // 32) * 32)
        k = self.payload_bits
        ph = torch.empty((batch_size, k), dtype=torch.uint8, pin_memory=True)
        dh = torch.empty((batch_size, k), dtype=torch.uint8, pin_memory=True)
        main = torch.cuda.current_stream()
        copy = L.side_stream("run_batch_d2h")
        for lo in range(0, batch_size, chunk):
            hi = min(batch_size, lo + chunk)
            p, d = self.run_batch_device(ebno_db, hi - lo, rng, lo)
            copy.wait_stream(main)
            with torch.cuda.stream(copy):
                ph[lo:hi].copy_(p, non_blocking=True)
                dh[lo:hi].copy_(d, non_blocking=True)
            p.record_stream(copy)
            d.record_stream(copy)
        copy.synchronize()
        return ph.numpy(), dh.numpy()

    def run_batch_counts(self, ebno_db: float, batch_size: int, rng: RngStream, counts=None):
        """Enqueue one batch and accumulate (bit_errors, block_errors) into the
        device int64[2] `counts` without any host synchronisation."""
        if counts is None:
            counts = L.zeros((2,), "int64")
        if self.family != "none" and (self.decoder_mode == "fast" or self.qc_exact):
            # decoder with derate, hard decision and error counting fused
            payload, llr = self._llr(ebno_db, batch_size, rng)
            qc_decode(llr, self.ldpc, self.bp_iter, self.bp_variant, self.bp_scale,
                      early_stop=self.bp_early_stop, ref_bits=payload, want_hard=False, counts=counts,
                      precision="exact" if self.decoder_mode == "exact" else self.precision)
            return counts
        p, d = self.run_batch_device(ebno_db, batch_size, rng)
        L.call("ls_count_errors", L.ptr(p), L.ptr(d), p.shape[0], p.shape[1], L.ptr(counts), L.stream_ptr())
        return counts


def build_pipeline(cfg: SimConfig) -> Pipeline:
    return Pipeline(cfg)


def _dist():
    try:
        import torch.distributed as dist
    except ImportError:  # pragma: no cover
        return None
    return dist if dist.is_available() and dist.is_initialized() else None


def _truncate(counts, target):
    """Deterministic stop (sweep.py:454-464): keep batches up to the first index
    whose cumulative block errors reach the target."""
    cum = 0
    for i, (_, blk) in enumerate(counts):
        cum += blk
        if cum >= target:
            return counts[: i + 1], True
    return counts, False


def sweep_points(cfg: SimConfig, payload_bits: int, eval_batch, dist=None, batches_per_rank: int = 1,
                 zeros=None) -> list:
    """The sweep loop of run_sweep (sweep.py:426-476), device-agnostic.

    eval_batch(snr_idx, ebno_db, batch_idx, out) accumulates that batch's
    (bit_errors, block_errors) into the int64[2] tensor `out`.  With a
    torch.distributed group, wave slot i goes to rank i % world; one
    all_gather per wave exchanges the counters.
    """
    import torch

    rank = dist.get_rank() if dist else 0
    world = dist.get_world_size() if dist else 1
    per = max(1, int(batches_per_rank))
    zeros = zeros or (lambda shape: torch.zeros(shape, dtype=torch.int64))
    points = []
    consecutive_zero = 0
    for snr_idx, ebno_db in enumerate(cfg.snr_points):
        start = time.perf_counter()
        if consecutive_zero >= 2:
            points.append(SnrPointResult(ebno_db, 0, 0, 0, 0, 0, "early-exit", 0.0))
            continue
        counts = []
        stop_reason = "max-batches"
        nxt = 0
        while nxt < cfg.max_batches_per_point:
            wave = list(range(nxt, min(nxt + world * per, cfg.max_batches_per_point)))
            local = zeros((per, 2))
            for i, bidx in enumerate(wave):
                if i % world == rank:
                    eval_batch(snr_idx, ebno_db, bidx, local[i // world])
            if dist:
                # NCCL gathers the device counters in place; gloo (CPU test
                # groups, or ranks sharing one GPU) needs host tensors
                src = local if dist.get_backend() == "nccl" else local.cpu()
                gathered = [torch.zeros_like(src) for _ in range(world)]
                dist.all_gather(gathered, src)
                allc = torch.stack(gathered).cpu()  # [world, per, 2]
            else:
                allc = local.cpu().unsqueeze(0)
            for i, _ in enumerate(wave):
                e = allc[i % world, i // world].tolist()
                counts.append((int(e[0]), int(e[1])))
            nxt = wave[-1] + 1
            counts, hit = _truncate(counts, cfg.target_block_errors)
            if hit:
                stop_reason = "target-errors"
                break
        bit_errors = sum(c[0] for c in counts)
        block_errors = sum(c[1] for c in counts)
        blocks = len(counts) * cfg.batch_size
        consecutive_zero = consecutive_zero + 1 if block_errors == 0 else 0
        points.append(SnrPointResult(ebno_db, blocks * payload_bits, bit_errors, blocks, block_errors,
                                     len(counts), stop_reason, time.perf_counter() - start))
    return points


def run_sweep(cfg: SimConfig, num_workers: int = 1, batches_per_rank: int = 1) -> SweepResult:
    """Eb/N0 sweep with error-count stopping and early exit (sweep.py:411-476).

    As in the reference, batches run in waves of `num_workers` before each
    stopping check (sweep.py:438-453): here a wave is enqueued on the GPU
    without host synchronisation, `ceil(num_workers / ranks)` batches per
    rank (or `batches_per_rank` if larger), and torch.distributed ranks (one
    per GPU) split it.  Statistics are identical for any worker or rank
    count (the prefix-truncation stop rule).
    """
    pipeline = build_pipeline(cfg)
    dist = _dist()
    world = dist.get_world_size() if dist else 1
    batches_per_rank = max(int(batches_per_rank), -(-max(1, int(num_workers)) // world))

    def eval_batch(snr_idx, ebno_db, bidx, out):
        rng = RngStream(cfg.seed, ((snr_idx + 1) << 32) | (bidx + 1))
        pipeline.run_batch_counts(ebno_db, cfg.batch_size, rng, counts=out)

    pts = sweep_points(cfg, pipeline.payload_bits, eval_batch, dist, batches_per_rank,
                       zeros=lambda shape: L.zeros(shape, "int64"))
    return SweepResult(config=cfg, points=pts)


def format_csv(result: SweepResult) -> str:
    """sweep.py:479-490: fixed columns, repr floats, '.' decimal."""
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(CSV_COLUMNS)
    for p in result.points:
        w.writerow([repr(p.ebno_db), p.bits, p.bit_errors, repr(p.ber), p.blocks, p.block_errors,
                    repr(p.bler), p.batches, p.stop_reason, repr(p.elapsed_s)])
    return buf.getvalue()


def write_csv(result: SweepResult, path) -> None:
    text = format_csv(result)
    try:
        with open(path, "w", encoding="ascii", newline="") as f:
            f.write(text)
    except OSError as exc:
        raise IOError(f"cannot write CSV to {path}: {exc}") from exc


def read_csv(path) -> list:
    out = []
    with open(path, "r", encoding="ascii", newline="") as f:
        reader = csv.DictReader(f)
        if tuple(reader.fieldnames or ()) != CSV_COLUMNS:
            raise ValueError(f"unexpected CSV columns: {reader.fieldnames}")
        for row in reader:
            out.append({k: (v if k == "stop_reason" else
                            float(v) if k in ("ebno_db", "ber", "bler", "elapsed_s") else int(v))
                        for k, v in row.items()})
    return out
