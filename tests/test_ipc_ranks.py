"""Cross-process ranks (tsd_ipc_*): two processes, one rank each, sharing
cuda:0, exchange CUDA IPC handles through a gloo process group and run MERLIN
and a range query with the fused peer-store transport (kills, row maxima and
exact-nn keys stored into every rank's arrays, event barriers between the
processes).  The records must equal the single-process ones bit for bit —
the same check bench.py's multi-GPU run relies on."""
import json
import os
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import paper_2304_01660_b200 as P
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x = P.gen_randomwalk(3000, 2024)
    e = P.Engine(0)
    e.set_series(x)
    h = e.ipc_export(len(x))
    hs = [None] * world
    dist.all_gather_object(hs, h)
    name = f"/tsd_test_{port}"
    if rank == 0:
        e.ipc_join(0, world, hs, name)
    dist.barrier()
    if rank != 0:
        e.ipc_join(rank, world, hs, name)
    dist.barrier()
    rep = e.merlin_full(8, 24, top_k=2, seglen=128)
    rng = e.pardrag(16, 60.0, 64)
    c = e.counters()
    res = {"recs": {str(m): [[int(r["index"]), float(r["nn_dist_sq"]).hex()] for r in v]
                    for m, v in rep.per_length.items()},
           "final_r": [float(v).hex() for v in rep.final_r], "retries": rep.retries.tolist(),
           "range": [[int(r["index"]), float(r["nn_dist_sq"]).hex()] for r in rng], "cells": int(c["cells"])}
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
        json.dump(res, f)
    dist.barrier()
    e.close()
    dist.destroy_process_group()


def test_two_processes_share_one_gpu(engine, tmp_path):
    import torch.multiprocessing as mp

    import paper_2304_01660_b200 as P
    world = 2
    mp.start_processes(worker, args=(world, free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    x = P.gen_randomwalk(3000, 2024)
    engine.set_series(x)
    rep = engine.merlin_full(8, 24, top_k=2, seglen=128)
    rng = engine.pardrag(16, 60.0, 64)
    want = {str(m): [[int(r["index"]), float(r["nn_dist_sq"]).hex()] for r in v] for m, v in rep.per_length.items()}
    res = [json.load(open(tmp_path / f"rank{r}.json")) for r in range(world)]
    for r in res:
        assert r["recs"] == want
        assert r["final_r"] == [float(v).hex() for v in rep.final_r] and r["retries"] == rep.retries.tolist()
        assert r["range"] == [[int(q["index"]), float(q["nn_dist_sq"]).hex()] for q in rng]
    assert all(r["cells"] > 0 for r in res)  # both ranks swept tiles
