"""Wall-clock per call of the host-buffer entry points (ldpc5g_decode with
pinned host LLRs; Pipeline.run_batch) and of the exact decoder."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2203_11854_b200 as lb  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
cfg = lb.SimConfig.from_dict({"code": {"family": "ldpc5g", "k": 8448, "n": 16896,
                                       "decoder": {"variant": "min-sum", "mode": "fast", "early_stop": False}},
                              "modulation": {"kind": "qam", "bits_per_symbol": 4},
                              "sweep": {"ebno_db": [6.0], "batch_size": B}})
pipe = lb.Pipeline(cfg)
_, llr = pipe._llr(6.0, B, lb.RngStream(1, 2))
host = torch.empty(llr.shape, dtype=torch.float32, pin_memory=True)
host.copy_(llr)
torch.cuda.synchronize()
for i in range(5):
    t = time.perf_counter()
    dec = lb.ldpc5g_decode(host, pipe.ldpc, 20, "min-sum", mode="fast", early_stop=False)
    torch.cuda.synchronize()
    print(f"decode_host call {i}: {(time.perf_counter() - t) * 1e3:.1f} ms")
for i in range(4):
    t = time.perf_counter()
    p, d = pipe.run_batch(6.0, B, lb.RngStream(1, 10 + i))
    print(f"run_batch call {i}: {(time.perf_counter() - t) * 1e3:.1f} ms")
small = llr[:1024].contiguous()
for i in range(4):
    torch.cuda.synchronize()
    t = time.perf_counter()
    lb.ldpc5g_decode(small, pipe.ldpc, 20, "min-sum", mode="exact", early_stop=False, device=True)
    torch.cuda.synchronize()
    print(f"exact 1024 call {i}: {(time.perf_counter() - t) * 1e3:.1f} ms")
