"""World-size-2 CPU tests (gloo) of the multi-process plumbing used by the NCCL path:
unique-id exchange, rank partitioning, and the block semantics of the global transpose
(emulated with point-to-point messages: send[d] -> recv[src], the ncclAlltoAll contract), checked end to end against numpy.fft.fft2."""
import os
import socket
import tempfile

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2004_09883_b200 as fb
    # 1. unique-id exchange (rank 0 creates it)
    uid = fb.exchange_unique_id(rank, world, lambda: bytes(range(128)))
    assert uid == bytes(range(128))
    # 2. slab forward with a real all_to_all over gloo
    n0, n1 = 32, 16
    rng = np.random.default_rng(7)
    x = rng.standard_normal((n0, n1)) + 1j * rng.standard_normal((n0, n1))
    r0, r1 = fb.slab_rows(rank, world, n0)
    rows, cols = n0 // world, n1 // world
    y = np.fft.fft(x[r0:r1], axis=1)
    send = np.empty((world, rows, cols), dtype=np.complex128)
    for k in range(n1):
        send[k // cols, :, k % cols] = y[:, k]
    # gloo has no alltoall: emulate ncclAlltoAll's contract (block d of rank s -> recv[s] of
    # rank d) with point-to-point sends/receives
    send_t = [torch.from_numpy(send[d].copy()) for d in range(world)]
    recv_t = [torch.empty_like(send_t[0]) for _ in range(world)]
    reqs = []
    for peer in range(world):
        if peer == rank:
            recv_t[peer].copy_(send_t[peer])
        else:
            reqs.append(dist.isend(send_t[peer], dst=peer))
            reqs.append(dist.irecv(recv_t[peer], src=peer))
    for q in reqs:
        q.wait()
    strip = np.concatenate([t.numpy() for t in recv_t], axis=0)
    ycols = np.fft.fft(strip, axis=0)
    c0, c1 = fb.slab_cols(rank, world, n1)
    ok = np.allclose(ycols, np.fft.fft2(x)[:, c0:c1], atol=1e-9)
    # 3. max-over-ranks timing reduction as in bench.py
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ok = ok and t.item() == float(world)
    open(os.path.join(outdir, f"r{rank}"), "w").write("ok" if ok else "bad")
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2():
    world = 2
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d), nprocs=world, join=True)
        assert all(open(os.path.join(d, f"r{r}")).read() == "ok" for r in range(world))
