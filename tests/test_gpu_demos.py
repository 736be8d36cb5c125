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


def test_waterfall_demo_sweep_matches_reference():
    """demos/ldpc_waterfall.py (the Listing-1 sweep: k=500 n=1000 sum-product,
    16-QAM max-log, 3-7 dB, error-count stop) through this package's
    run_sweep in exact mode, against the reference's own run_sweep result
    (tests/golden/demo_waterfall.json, tests/golden/make_demo_golden.py)."""
    import json
    import os

    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "demo_waterfall.json")))
    res = lb.run_sweep(lb.SimConfig.from_dict(gold["config"]), num_workers=4)
    assert len(res.points) == len(gold["points"])
    for p, g in zip(res.points, gold["points"]):
        assert (p.ebno_db, p.bits, p.blocks, p.batches, p.stop_reason) == (
            g["ebno_db"], g["bits"], g["blocks"], g["batches"], g["stop_reason"])
        assert (p.bit_errors, p.block_errors) == (g["bit_errors"], g["block_errors"])
