"""Debug: single context vs two IPC ranks on one device, one pardrag call."""
import os
import socket
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def worker(rank, world, port, m, r_sq):
    import torch.distributed as dist

    import paper_2304_01660_b200 as P
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x = P.gen_randomwalk(3000, 2024)
    e = P.Engine(0)
    e.set_series(x)
    hs = [None] * world
    dist.all_gather_object(hs, e.ipc_export(len(x)))
    name = f"/tsd_dbg_{port}"
    if rank == 0:
        e.ipc_join(0, world, hs, name)
    dist.barrier()
    if rank != 0:
        e.ipc_join(rank, world, hs, name)
    dist.barrier()
    if m == 0:
        rep = e.merlin_full(8, 24, top_k=2, seglen=128)
        for mm in (15, 16, 17, 18):
            print(f"rank {rank} m={mm}: {[(int(g['index']), float(g['nn_dist_sq'])) for g in rep.per_length[mm]]}",
                  flush=True)
    else:
        got = e.pardrag(m, r_sq, 64)
        print(f"rank {rank}: {len(got)} survivors, tail {[(int(g['index']), float(g['nn_dist_sq'])) for g in got[:4]]}",
              flush=True)
    dist.barrier()
    e.close()


if __name__ == "__main__":
    import torch.multiprocessing as mp

    import paper_2304_01660_b200 as P
    m, r_sq = int(sys.argv[1]), float(sys.argv[2])
    x = P.gen_randomwalk(3000, 2024)
    e = P.Engine(0)
    e.set_series(x)
    if m == 0:
        rep = e.merlin_full(8, 24, top_k=2, seglen=128)
        for mm in (15, 16, 17, 18):
            print(f"single m={mm}: {[(int(g['index']), float(g['nn_dist_sq'])) for g in rep.per_length[mm]]}")
    else:
        got = e.pardrag(m, r_sq, 64)
        print(f"single: {len(got)} survivors, head {[(int(g['index']), float(g['nn_dist_sq'])) for g in got[:4]]}")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.start_processes(worker, args=(2, port, m, r_sq), nprocs=2, join=True, start_method="spawn")
