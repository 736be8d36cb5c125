"""B200-native (sm_100a) drop-in for the linksim coded-link hot path.

Mirrors the reference's block API (linksim/__init__.py:11-32) for the
batched Monte-Carlo chain binary_source -> ldpc5g_encode -> map_bits ->
awgn -> demap_app|demap_maxlog -> ldpc5g_decode/bp_decode -> count_errors,
driven by Pipeline.run_batch / run_sweep.  All array work runs in the CUDA
library liblinksim_b200.so (include/linksim_b200.h); there is no CPU
fallback.
"""
from .alist import AlistParseError, ParityCheckMatrix, parse_alist, to_alist
from .channel import awgn, complex_gaussian
from .core import (LLR_MAX, RngStream, binary_source, compute_ber, compute_bler, count_errors,
                   ebnodb2no, hard_decide)
from .ldpc import (BP_VARIANTS, LIFTING_SIZES, LdpcCode5G, bp_decode, exit_mutual_information,
                   ldpc5g_decode, ldpc5g_encode, qc_decode)
from .mapping import Constellation, demap_app, demap_maxlog, map_bits
from .sweep import (ConfigError, Pipeline, SimConfig, SnrPointResult, SweepResult, format_csv,
                    read_csv, run_sweep, write_csv)

__version__ = "0.1.0"
__all__ = [
    "ParityCheckMatrix", "AlistParseError", "parse_alist", "to_alist", "awgn", "complex_gaussian", "LLR_MAX", "RngStream", "binary_source",
    "compute_ber", "compute_bler", "count_errors", "ebnodb2no", "hard_decide", "BP_VARIANTS",
    "LIFTING_SIZES", "LdpcCode5G", "bp_decode", "exit_mutual_information", "ldpc5g_decode",
    "ldpc5g_encode", "qc_decode", "Constellation", "demap_app", "demap_maxlog", "map_bits",
    "ConfigError", "Pipeline", "SimConfig", "SnrPointResult", "SweepResult", "format_csv",
    "read_csv", "run_sweep", "write_csv",
]
