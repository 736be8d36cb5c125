"""CPU tests of the host side: the C-ABI library loads and exports every
declared symbol, the restated base graphs, code construction, config
validation, the CSV contract and the multi-rank sweep logic (gloo)."""
import os
import re
import socket
import ctypes

import numpy as np
import pytest

import paper_2203_11854_b200 as lb
from paper_2203_11854_b200 import _lib as L
from paper_2203_11854_b200.basegraph import base_graph
from paper_2203_11854_b200.sweep import SimConfig, SnrPointResult, SweepResult, sweep_points
from oracle import linksim_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "linksim_b200.h")).read()
    names = sorted(set(re.findall(r"\b(ls_[a-z0-9_]+)\s*\(", hdr)))
    assert len(names) >= 15
    lib = L.lib()
    for nm in names:
        assert hasattr(lib, nm), nm
        # every entry point has typed ctypes argtypes in the Python binding
        assert nm == "ls_last_error" or nm in L._SIGS, nm
    assert lib.ls_version() >= 1


def test_library_rejects_bad_arguments_without_gpu():
    lib = L.lib()
    h = ctypes.c_void_p()
    ent = np.zeros((1, 3), np.int32)
    rc = lib.ls_code_create(3, 8, 10, 20, 1, 1, 1, ent.ctypes.data, 1, ctypes.byref(h))
    assert rc == L.LS_EINVAL and b"unknown base graph" in lib.ls_last_error()
    rc = lib.ls_code_create(1, 8, 30, 20, 46, 68, 22, ent.ctypes.data, 1, ctypes.byref(h))
    assert rc == L.LS_EINVAL and b"need 0 < k < n" in lib.ls_last_error()


@pytest.mark.parametrize("bg", [1, 2])
def test_base_graph_restatement_matches_reference_tables(golden, bg):
    z = golden("base_graphs")
    ent, mb, nb, kb = base_graph(bg)
    assert np.array_equal(ent, z[f"bg{bg}"])
    assert (mb, nb, kb) == tuple(int(x) for x in z[f"bg{bg}_dims"])


@pytest.mark.parametrize("k,n", [(500, 1000), (100, 300), (256, 512), (8448, 16896), (4096, 8192),
                                 (4096, 12288), (256, 1536), (1, 3), (40, 200), (8448, 25344)])
def test_code_dimensions_and_rate_matching(k, n):
    c = lb.LdpcCode5G(k, n)
    o = O.Code(k, n)
    assert (c.base_graph, c.z) == (o.bg, o.z)
    assert np.array_equal(c.transmit_idx, o.transmit_idx)
    assert (c.k_full, c.n_full, c.m_full) == (o.k_full, o.n_full, o.m_full)


def test_dimension_selection_known_answers():
    assert (lb.LdpcCode5G(500, 1000).base_graph, lb.LdpcCode5G(500, 1000).z) == (1, 24)
    assert (lb.LdpcCode5G(100, 300).base_graph, lb.LdpcCode5G(100, 300).z) == (2, 10)
    with pytest.raises(ValueError):
        lb.LdpcCode5G(100, 90)
    with pytest.raises(ValueError):
        lb.LdpcCode5G(0, 100)


def test_lifted_pcm_matches_oracle_csr():
    c = lb.LdpcCode5G(256, 512)
    o = O.code(256, 512)
    ptr, var = c.pcm.csr()
    assert np.array_equal(ptr, o._csr[0]) and np.array_equal(var, o._csr[1])


def test_ebnodb2no_known_values():
    assert lb.ebnodb2no(10.0, 4, 0.5) == pytest.approx(0.05)
    with pytest.raises(ValueError):
        lb.ebnodb2no(1.0, 0, 0.5)
    with pytest.raises(ValueError):
        lb.ebnodb2no(1.0, 2, 1.5)


BASE_CFG = {"code": {"family": "ldpc5g", "k": 256, "n": 512},
            "modulation": {"kind": "qam", "bits_per_symbol": 2},
            "sweep": {"ebno_db": [1.0, 2.0], "batch_size": 8}}


@pytest.mark.parametrize("patch,field", [
    ({"code": {"family": "turbo", "k": 10}}, "code.family"),
    ({"code": {"family": "ldpc5g", "k": 0, "n": 10}}, "code.k"),
    ({"code": {"family": "ldpc5g", "k": 10, "n": 5}}, "code.n"),
    ({"modulation": {"kind": "qam", "bits_per_symbol": 3}}, "modulation.bits_per_symbol"),
    ({"modulation": {"kind": "ask", "bits_per_symbol": 2}}, "modulation.kind"),
    ({"sweep": {"ebno_db": [2.0, 1.0]}}, "sweep.ebno_db"),
    ({"sweep": {"ebno_db": []}}, "sweep.ebno_db"),
    ({"sweep": {"ebno_db": [1.0], "batch_size": 0}}, "sweep.batch_size"),
    ({"precision": "half"}, "precision"),
    ({"code": {"family": "ldpc5g", "k": 256, "n": 512, "decoder": {"variant": "x"}}}, "code.decoder.variant"),
    ({"modulation": {"kind": "qam", "bits_per_symbol": 2, "demapper": "x"}}, "modulation.demapper"),
])
def test_config_errors_name_the_field(patch, field):
    raw = dict(BASE_CFG)
    raw.update(patch)
    with pytest.raises(lb.ConfigError) as ei:
        SimConfig.from_dict(raw)
    assert ei.value.field == field


def test_csv_round_trip(tmp_path):
    cfg = SimConfig.from_dict(BASE_CFG)
    res = SweepResult(cfg, [SnrPointResult(1.0, 2560, 3, 10, 1, 1, "max-batches", 0.25),
                            SnrPointResult(2.0, 0, 0, 0, 0, 0, "early-exit", 0.0)])
    p = tmp_path / "r.csv"
    lb.write_csv(res, p)
    rows = lb.read_csv(p)
    assert rows[0]["bits"] == 2560 and rows[0]["ber"] == 3 / 2560 and rows[1]["stop_reason"] == "early-exit"
    assert open(p).read().splitlines()[0] == ",".join(lb.sweep.CSV_COLUMNS)


def _fake_eval(snr_idx, ebno, bidx, out):
    # deterministic per (snr, batch) like the reference's RNG keying
    g = np.random.default_rng(1000 * snr_idx + bidx)
    blk = int(g.integers(0, 4)) if snr_idx < 2 else 0
    out[0] += blk * 3 + int(g.integers(0, 2))
    out[1] += blk


def _cfg_for_sweep():
    return SimConfig.from_dict({**BASE_CFG, "sweep": {"ebno_db": [0.0, 1.0, 2.0, 3.0, 4.0], "batch_size": 8,
                                                      "target_block_errors": 9, "max_batches_per_point": 7}})


def _worker(rank, world, port, q):
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    pts = sweep_points(_cfg_for_sweep(), 256, _fake_eval, dist, batches_per_rank=2)
    q.put((rank, [(p.bits, p.bit_errors, p.blocks, p.block_errors, p.batches, p.stop_reason) for p in pts]))
    dist.destroy_process_group()


def test_sweep_points_identical_for_any_rank_count_gloo():
    import torch.multiprocessing as mp

    ref = sweep_points(_cfg_for_sweep(), 256, _fake_eval, None, batches_per_rank=1)
    ref = [(p.bits, p.bit_errors, p.blocks, p.block_errors, p.batches, p.stop_reason) for p in ref]
    assert [r[5] for r in ref][:2] == ["target-errors", "target-errors"]
    assert [r[5] for r in ref][-1] == "early-exit"
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for _, pts in got:
        assert pts == ref
