"""Host-LLR decode (ldpc5g_decode with pinned host f32 LLRs -> host bits) at
several pipeline chunk sizes: python tools/prof_hostdecode.py."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2203_11854_b200 as lb  # noqa: E402
from paper_2203_11854_b200 import ldpc  # noqa: E402

B = 65536
cfg = lb.SimConfig.from_dict({"code": {"family": "ldpc5g", "k": 8448, "n": 16896, "decoder": {"mode": "fast"}},
                              "modulation": {"kind": "qam", "bits_per_symbol": 4},
                              "sweep": {"ebno_db": [6.0], "batch_size": B}})
pipe = lb.Pipeline(cfg)
_, llr = pipe._llr(6.0, B, lb.RngStream(1, 2))
host = torch.empty(llr.shape, dtype=torch.float32, pin_memory=True)
host.copy_(llr)
del llr
for chunk in (2048, 2048, 2048, 8192, 2048):
    for _ in range(2):
        ldpc._decode_host_pipelined(host, pipe.ldpc, 20, "min-sum", 0.75, False, "fp16x2", chunk=chunk)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        ldpc._decode_host_pipelined(host, pipe.ldpc, 20, "min-sum", 0.75, False, "fp16x2", chunk=chunk)
    torch.cuda.synchronize()
    el = (time.perf_counter() - t) / 3
    print(f"chunk {chunk:6d}: {el * 1e3:7.1f} ms/step, {B * 8448 / el / 1e9:.2f} Gbit/s")
