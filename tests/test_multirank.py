"""World-size-2 (gloo, CPU) checks of the multi-GPU design: tiles of the
distance matrix dealt cyclically over ranks, kill flags AND-reduced
(all_reduce MIN on uint8), exact minima MIN-reduced.  The per-rank work here is
a numpy model of one tile (exact z-normalised distances from the oracle's
definition), so the test exercises the sharding rule and the reduction
semantics the engine uses (engine.cu: run_scan's cyclic deal, allreduce_* after
every scan) without a GPU: the sharded result must equal the single-rank
range-discord set {c : nn(c)^2 >= r^2} with identical nn."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

KW = 64  # model tile width (diagonals)


def znorm_rows(x, m):
    N = len(x) - m + 1
    w = np.lib.stride_tricks.sliding_window_view(x, m)[:N]
    mu = w.mean(axis=1, keepdims=True)
    sd = w.std(axis=1, keepdims=True)
    return (w - mu) / sd


def tiles_for(N, m, rows=32):
    """Full-row tiles (r0, rows, k0, dir) like engine.cu full_row_tiles: both
    sides of every row block, chunk-major."""
    out = []
    groups = [(a, min(N, a + rows) - 1) for a in range(0, N, rows)]
    npos = [max(0, -(-(N - a - m) // KW)) for a, _ in groups]
    nneg = [max(0, -(-(b - m + 1) // KW)) for _, b in groups]
    for i in range(max(npos + nneg)):
        for g, (a, b) in enumerate(groups):
            if i < npos[g]:
                out.append((a, b - a + 1, m + i * KW, +1))
            if i < nneg[g]:
                out.append((a, b - a + 1, -m - (i + 1) * KW + 1, -1))
    return out


def tile_cells(tile, N):
    r0, rows, k0, d = tile
    for s in range(rows):
        c = r0 + s
        for k in range(k0, k0 + KW):
            q = c + k
            if 0 <= q < N:
                yield c, q


def sharded_range(rank, world, x, m, r_sq):
    Z = znorm_rows(x, m)
    N = len(Z)
    tl = tiles_for(N, m)
    mine = tl[rank::world]  # cyclic deal, as run_scan does
    alive = torch.ones(N, dtype=torch.uint8)
    nn = torch.full((N,), float("inf"), dtype=torch.float64)
    for t in mine:
        for c, q in tile_cells(t, N):
            d = float(np.sum((Z[c] - Z[q]) ** 2))
            if d < r_sq:
                alive[c] = 0
            nn[c] = min(float(nn[c]), d)
    if world > 1:
        dist.all_reduce(alive, op=dist.ReduceOp.MIN)  # AND of {0,1} flags
        dist.all_reduce(nn, op=dist.ReduceOp.MIN)
    idx = torch.nonzero(alive).flatten().numpy()
    return idx, nn.numpy()[idx], len(tl), len(mine)


def _worker(rank, world, port, x, m, r_sq, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    idx, nn, nt, nmine = sharded_range(rank, world, x, m, r_sq)
    tot = torch.tensor([nmine])
    dist.all_reduce(tot)
    if rank == 0:
        q.put((idx.tolist(), nn.tolist(), nt, int(tot.item())))
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

    idx1, nn1, nt, _ = sharded_range(0, 1, x, m, r_sq)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, x, m, r_sq, q)) for r in range(2)]
    for p in procs:
        p.start()
    idx2, nn2, nt2, covered = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # the cyclic deal covers every tile exactly once
    assert nt2 == nt and covered == nt
    # identical survivors at 1 and 2 ranks, equal to the oracle's range set
    assert list(idx1) == idx2 == sorted(int(i) - 1 for i in exp["index"])
    assert np.allclose(nn1, nn2, rtol=0, atol=1e-9)
    got = dict(zip(idx2, nn2))
    for r in exp:
        assert abs(got[int(r["index"]) - 1] - r["nn_dist_sq"]) <= 1e-9 * max(1.0, r["nn_dist_sq"])
