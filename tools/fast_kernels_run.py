"""One fixed-iteration launch of the fp16x2 (k_qc_fast_h2w) and the fp32
full-graph (k_qc_exact<..., float>) decoders at the bench size, for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2203_11854_b200 as lb  # noqa: E402


class A:
    seed, iters, ebno, batch, variant = 42, 20, 6.0, 65536, "min-sum"


pipe = bench._fast_pipe(A, "min-sum")
payload, llr = pipe._llr(6.0, A.batch, lb.RngStream(42, 700))
for prec, prune in (("fp16x2", True), ("fp32-full", False)):
    lb.qc_decode(llr, pipe.ldpc, 20, "min-sum", 0.75, early_stop=False, ref_bits=payload, want_hard=False,
                 precision=prec, prune=prune)
torch.cuda.synchronize()
print("done")
