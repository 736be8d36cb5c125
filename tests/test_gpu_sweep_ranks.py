"""run_sweep on the REAL pipeline across ranks.

The reference's run_sweep result for a small config-1 sweep is a golden
(tests/golden/sweep_c1.npz, minted by make_goldens.py from the unmodified
reference, deterministic in (config, seed) for any worker count).  The
exact-mode GPU sweep must reproduce it point for point -- counts, batches,
stop reasons -- with one rank, and with two torch.distributed ranks whose
per-wave counters are exchanged by all_gather.  Both ranks share cuda:0 here
(gloo carries the counters: the box has one GPU); the ranks never wait on
each other's kernels, only on the host-side collective, so this is the
multi-rank code path of run_sweep unchanged.
"""
import json
import os
import socket
import tempfile

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - collected on CPU boxes
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2203_11854_b200 as lb  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "sweep_c1.npz")


def _golden():
    d = np.load(GOLD)
    return json.loads(str(d["config"])), d


def _points(res):
    return [(p.ebno_db, p.bits, p.bit_errors, p.blocks, p.block_errors, p.batches, p.stop_reason)
            for p in res.points]


def _gold_points(d):
    return [(float(d["ebno"][i]), int(d["bits"][i]), int(d["bit_errors"][i]), int(d["blocks"][i]),
             int(d["block_errors"][i]), int(d["batches"][i]), str(d["stop_reason"][i]))
            for i in range(len(d["ebno"]))]


@pytest.mark.parametrize("workers", [1, 3])
def test_run_sweep_one_rank_equals_reference(workers):
    cfg, d = _golden()
    res = lb.run_sweep(lb.SimConfig.from_dict(cfg), num_workers=workers)
    assert _points(res) == _gold_points(d)
    assert lb.format_csv(res).splitlines()[0] == str(d["csv_header"])


def _rank_main(rank, world, port, out_path, workers):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg, _ = _golden()
        res = lb.run_sweep(lb.SimConfig.from_dict(cfg), num_workers=workers)
        if rank == 0:
            with open(out_path, "w") as f:
                json.dump(_points(res), f)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("workers", [2, 5])
def test_run_sweep_two_ranks_equals_reference(workers):
    import torch.multiprocessing as mp

    _, d = _golden()
    with tempfile.TemporaryDirectory() as tmp:
        out = os.path.join(tmp, "r0.json")
        mp.spawn(_rank_main, args=(2, _free_port(), out, workers), nprocs=2, join=True)
        got = [tuple(x) for x in json.load(open(out))]
    assert got == _gold_points(d)
