"""Multi-process (world_size 2, gloo, CPU) tests of the sharding host logic and of the a9
allgather: the per-rank records (header format, tests/xchg_ref.py) gathered in ONE collective give
the single-process batch boundaries and totals.  The per-rank compute
is the CPU oracle here (no GPU in this container); on a B200 box the same host path wraps the
CUDA library (bench.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2409_14961_b200 import distributed as D
from tests import xchg_ref as X


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import workloads as W
        inp, out, slo, cfg = W.c3(5, n=60_000)
        cfg = cfg.replace(window=7_000)
        qb = D.query_begins(len(inp), cfg.window, world)
        a, z = qb[rank], qb[rank + 1]
        order, offs, m, cost = oracle.schedule(inp[a:z], out[a:z], slo[a:z], cfg)
        pb, tot = oracle.stats(inp[a:z], out[a:z], slo[a:z], cfg, order, offs)
        lat = int((pb["size"].astype(object) * pb["completion_us"].astype(object)).sum()) if len(pb) else 0
        # the a9 record in the header's format (on the GPU the library writes it: uellm_exchange_pack)
        n_max = max(y - x for x, y in zip(qb[:-1], qb[1:]))
        rec = torch.from_numpy(X.make_record(tot, lat, offs, z - a, n_max))
        gathered = torch.zeros(world * rec.numel(), dtype=torch.uint8)
        dist.all_gather(list(gathered.view(world, -1).unbind(0)), rec)      # ONE collective
        offs_all, comb = X.combine(gathered.view(world, -1).numpy(), qb)
        if rank == 0:
            q.put((comb, offs_all))
    finally:
        dist.destroy_process_group()


def test_window_blocks_partition():
    for nwin in (0, 1, 5, 100, 101):
        for world in (1, 2, 3, 8):
            blocks = [D.window_block(nwin, world, r) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == nwin
            assert all(b[1] == c[0] for b, c in zip(blocks, blocks[1:]))
            sizes = [b[1] - b[0] for b in blocks]
            assert max(sizes) - min(sizes) <= 1


def test_query_ranges_align_to_windows():
    n, wl = 1_000_003, 100_000
    rs = [D.query_range(n, wl, 8, r) for r in range(8)]
    assert rs[0][0] == 0 and rs[-1][1] == n
    assert all(a % wl == 0 for a, _ in rs)


def test_allgather_world2_equals_single_process():
    import oracle
    import workloads as W
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    comb, offs_all = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    inp, out, slo, cfg = W.c3(5, n=60_000)
    cfg = cfg.replace(window=7_000)
    order, offs, m, cost = oracle.schedule(inp, out, slo, cfg)
    _, tot = oracle.stats(inp, out, slo, cfg, order, offs)
    for f in X.TOTAL_FIELDS:
        assert comb[f] == tot[f], f
    assert comb["dp_cost"] == cost
    assert np.array_equal(offs_all, offs.astype(np.int64))      # global batch boundaries
    assert comb["mean_latency_s"] == pytest.approx(tot["mean_latency_s"], rel=1e-12)
    assert comb["throughput_tok_s"] == pytest.approx(tot["throughput_tok_s"], rel=1e-12)


def test_record_size_matches_library():
    """The library's record size (uellm_exchange_bytes, a host function) is the header's layout."""
    from paper_2409_14961_b200 import uellm as U
    for n_max in (0, 1, 31, 32, 33, 1000, 12_500_000):
        assert U.exchange_bytes(n_max) == X.record_bytes(n_max)
    assert U.TOTALS_BYTES == 128


def test_query_begins():
    qb = D.query_begins(1_000_003, 100_000, 8)
    assert qb[0] == 0 and qb[-1] == 1_000_003 and len(qb) == 9
    assert all(x <= y for x, y in zip(qb, qb[1:]))
    assert D.query_begins(5, 10, 4) == [0, 0, 0, 0, 5]          # one window, three empty ranks
