"""Multi-process (world_size 2, gloo, CPU) tests of the sharding host logic and of the a9
allgather: the combined per-rank totals equal the single-process result.  The per-rank compute
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
        a, z = D.query_range(len(inp), cfg.window, world, rank)
        order, offs, m, cost = oracle.schedule(inp[a:z], out[a:z], slo[a:z], cfg)
        _, tot = oracle.stats(inp[a:z], out[a:z], slo[a:z], cfg, order, offs)
        g = D.all_gather_totals(D.pack_totals(tot, "cpu"))
        comb = D.combine_totals(g)
        # the a9 buffer proper: [totals | boundary bitmap of this rank's positions], padded to the
        # largest rank (on the GPU the library writes the bitmap, uellm_boundary_bitmap)
        ranges = [D.query_range(len(inp), cfg.window, world, r) for r in range(world)]
        n_max = max(b - a_ for a_, b in ranges)
        buf = torch.zeros(D.exchange_words(n_max), dtype=torch.int64)
        buf[:D.GATHER_WORDS] = D.pack_totals(tot, "cpu")
        bits = np.zeros(32 * D.bitmap_view(buf).numel(), np.uint8)
        bits[offs.astype(np.int64)] = 1
        D.bitmap_view(buf).copy_(torch.from_numpy(np.packbits(bits, bitorder="little").view(np.int32)))
        gx = D.all_gather_exchange(buf)
        offs_all = D.global_offsets(gx, ranges)
        comb2 = D.combine_totals(gx[:, :D.GATHER_WORDS])
        if rank == 0:
            q.put((comb, cost, offs_all, comb2))
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
    comb, _, offs_all, comb2 = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    inp, out, slo, cfg = W.c3(5, n=60_000)
    cfg = cfg.replace(window=7_000)
    order, offs, m, cost = oracle.schedule(inp, out, slo, cfg)
    _, tot = oracle.stats(inp, out, slo, cfg, order, offs)
    for f in D.TOTAL_FIELDS:
        assert comb[f] == tot[f], f
    assert comb["dp_cost"] == cost
    assert np.array_equal(offs_all, offs.astype(np.int64))      # global batch boundaries
    assert comb2 == comb
    assert comb["mean_latency_s"] == pytest.approx(tot["mean_latency_s"], rel=1e-12)
    assert comb["throughput_tok_s"] == pytest.approx(tot["throughput_tok_s"], rel=1e-12)


def test_pack_roundtrip():
    tot = {f: (i + 1) * 1234567 for i, f in enumerate(D.TOTAL_FIELDS)}
    tot["dp_cost"] = 2**63 + 5
    tot["mean_latency_s"] = 3.25
    tot["throughput_tok_s"] = 1e9 / 3
    v = D.pack_totals(tot, "cpu").view(1, -1)
    c = D.combine_totals(v)
    assert c["dp_cost"] == 2**63 + 5
    assert c["mean_latency_s"] == 3.25
