"""World-size-2 (gloo, CPU) checks of the multi-GPU design: tiles of the
distance matrix dealt cyclically over ranks, kill flags AND-reduced
(all_reduce MIN on uint8), exact minima MIN-reduced.

The tiles are the ENGINE'S OWN: every rank asks libtsdiscord_b200.so's host
planner (tsd_tile_plan, which runs the kernels' decoder from tile_space.cuh)
for the slots it owns in each launch of a try's tile spaces -- band 0 over
row blocks at the resident offset kA, a later band over groups, and the full
rows over groups -- so the test exercises the real cyclic deal (rank r fetches
slots r, r+world, ...) and the real tile geometry (1152 diagonals, both sides).
Only the per-cell arithmetic is a model (exact z-normalised distances from the
oracle's definition, in numpy): the sharded result must equal the single-rank
range-discord set {c : nn(c)^2 >= r^2} with identical nn, and the ranks' tiles
must partition the single-rank tile set."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

KW = 1152  # tile width (diagonals), common.cuh kW


def znorm_rows(x, m):
    N = len(x) - m + 1
    w = np.lib.stride_tricks.sliding_window_view(x, m)[:N]
    mu = w.mean(axis=1, keepdims=True)
    sd = w.std(axis=1, keepdims=True)
    return (w - mu) / sd


def engine_tiles(N, m, rank, world):
    """The tiles of one try's launches as the engine deals them to `rank`."""
    import paper_2304_01660_b200 as P
    L = 128
    kA = m + 7  # band 0 at a fixed offset >= m (MERLIN: kA = maxL)
    groups = [(a, min(N, a + 48) - 1) for a in range(0, N, 48)]
    out = []
    for t in P.tile_plan("seed", N, m, rank, world, L=L, kA=kA, nb=2):
        out.append(("seed",) + tuple(int(v) for v in t))
    for t in P.tile_plan("band", N, m, rank, world, K0=kA + KW, nb=1, groups=groups):
        out.append(("band",) + tuple(int(v) for v in t))
    for t in P.tile_plan("full", N, m, rank, world, groups=groups):
        out.append(("full",) + tuple(int(v) for v in t))
    return out


def tile_cells(tile, N, m):
    _, r0, rows, k0, d, _ = tile
    for s in range(rows):
        c = r0 + s
        for k in range(k0, k0 + KW):
            q = c + k
            if 0 <= q < N and abs(k) >= m:
                yield c, q


def sharded_range(rank, world, x, m, r_sq):
    Z = znorm_rows(x, m)
    N = len(Z)
    tl = engine_tiles(N, m, 0, 1)
    mine = engine_tiles(N, m, rank, world)  # the engine's cyclic deal of every launch
    alive = torch.ones(N, dtype=torch.uint8)
    nn = torch.full((N,), float("inf"), dtype=torch.float64)
    for t in mine:
        for c, q in tile_cells(t, N, m):
            d = float(np.sum((Z[c] - Z[q]) ** 2))
            if d < r_sq:
                alive[c] = 0
            nn[c] = min(float(nn[c]), d)
    if world > 1:
        dist.all_reduce(alive, op=dist.ReduceOp.MIN)  # AND of {0,1} flags
        dist.all_reduce(nn, op=dist.ReduceOp.MIN)
    idx = torch.nonzero(alive).flatten().numpy()
    return idx, nn.numpy()[idx], tl, mine


def _worker(rank, world, port, x, m, r_sq, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    idx, nn, tl, mine = sharded_range(rank, world, x, m, r_sq)
    every = [None] * world
    dist.all_gather_object(every, mine)
    if rank == 0:
        q.put((idx.tolist(), nn.tolist(), tl, every))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("seed,m,qtl", [(3, 8, 0.9), (4, 12, 0.5)])
def test_world2_equals_world1_and_oracle(oracle, seed, m, qtl):
    x = oracle.gen_randomwalk(360, seed)
    nn_ref = oracle.brute_force_nn(x, m)
    srt = np.sort(nn_ref)
    k = int(len(srt) * qtl)
    r_sq = float(0.5 * (srt[k] + srt[k + 1]))  # between two profile values: no arithmetic ties
    exp = oracle.range_discords(x, m, r_sq)

    idx1, nn1, tl, _ = sharded_range(0, 1, x, m, r_sq)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, x, m, r_sq, q)) for r in range(2)]
    for p in procs:
        p.start()
    idx2, nn2, tl2, every = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # the ranks' tiles partition the single-rank tile set (every tile exactly once)
    assert tl2 == tl
    assert sorted(every[0] + every[1]) == sorted(tl)
    assert not set(every[0]) & set(every[1]) and every[0] and every[1]
    # identical survivors at 1 and 2 ranks, equal to the oracle's range set
    assert list(idx1) == idx2 == sorted(int(i) - 1 for i in exp["index"])
    assert np.allclose(nn1, nn2, rtol=0, atol=1e-9)
    got = dict(zip(idx2, nn2))
    for r in exp:
        assert abs(got[int(r["index"]) - 1] - r["nn_dist_sq"]) <= 1e-9 * max(1.0, r["nn_dist_sq"])
