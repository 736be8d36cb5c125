"""The reference's hot-path demo (demos/exit_tracking.py:19-35: BP one
iteration count at a time plus the EXIT mutual information of the output
LLRs) run through this package's public API, against the oracle's
sum-product BP and MI on the same mother LLRs."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - collected on CPU boxes
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2203_11854_b200 as lb  # noqa: E402
from oracle import linksim_oracle as O  # noqa: E402


@pytest.mark.parametrize("ebno_db", [-1.0, 1.0, 3.0])
def test_exit_tracking_demo_trajectory(ebno_db):
    K, N, B = 100, 300, 64
    rng = lb.RngStream(31, 0).child(1)
    code = lb.LdpcCode5G(K, N)
    const = lb.Constellation("qam", 2)
    bits = lb.binary_source([B, K], rng.child(0))
    tx = lb.ldpc5g_encode(bits, code)
    x = lb.map_bits(tx, const)
    no = lb.ebnodb2no(ebno_db, 2, K / N)
    y = lb.awgn(x, no, rng.child(1))
    llr = lb.demap_app(y, no, const)
    mother = code.derate_match(llr)
    truth = code.encode_full(bits)
    oc = O.code(K, N)
    prev = -1.0
    for it in (1, 2, 4, 8, 16):
        llr_out, _ = lb.bp_decode(mother, code.pcm, num_iter=it, early_stop=False)
        mi = lb.exit_mutual_information(llr_out, truth)
        lo_o, _, _ = O.bp_decode_csr(np.asarray(mother, np.float64), *(oc._csr if hasattr(oc, "_csr") else oc.csr), oc.n_full, it, "sum-product",
                                     0.75, False)
        mi_o = O.exit_mutual_information(lo_o, np.asarray(truth))
        assert abs(mi - mi_o) < 1e-6
        assert 0.0 <= mi <= 1.0
        if ebno_db >= 1.0:
            assert mi >= prev - 1e-3  # the climb toward 1.0 above threshold
        prev = mi
