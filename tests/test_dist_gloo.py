"""World-size-2 CPU (gloo) tests of the row-sharded decomposition the NCCL
path implements (paper_1505_07570_b200/csrc/api_sketch.cpp
combined_gaussian_pipelined, dist.cpp):

* rows are split by rnla_shard_rows; each rank hashes its rows by GLOBAL
  index (row_offset = sum of lower ranks' counts, found by an allgather);
* the per-rank count-sketch partials sum (allreduce) to the single-process
  sketch;
* the Gaussian stage is split into canonical K-chunks of s/world buckets,
  chunk c is reduced onto owner rank c % world, the owner multiplies it, and
  an allreduce of the s2 x (d+1) partial products gives the full sketch.
The arithmetic runs in the CPU oracle; the GPU path is covered by the
-m gpu tests on one device.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1505_07570_b200 as rn
from oracle import oracle as orc


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, d, s, s2, seed, seed2, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(123)
        a = rng.standard_normal((n, d))
        b = rng.standard_normal(n)
        r0, r1 = rn.shard_rows(n, world, rank)
        # global row offset from every rank's local count (dist.cpp global_row_offset)
        counts = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(counts, torch.tensor([r1 - r0], dtype=torch.int64))
        off = int(sum(int(c.item()) for c in counts[:rank]))
        assert off == r0
        part = orc.count_sketch_rows(a[r0:r1], s, seed, extra=b[r0:r1], j0=off)
        # (1) allreduce of the count partials
        t = torch.from_numpy(part.copy())
        dist.all_reduce(t)
        full_mid = orc.count_sketch_rows(a, s, seed, extra=b)
        ok_mid = np.allclose(t.numpy(), full_mid, rtol=0, atol=1e-12)
        # (2) chunked Gaussian stage with per-chunk reduce to the owner
        g = orc.gaussian_matrix(s, s2, seed2) / np.sqrt(s2)
        kc = (s + world - 1) // world
        acc = np.zeros((s2, d + 1))
        mid = torch.from_numpy(part.copy())
        for c, b0 in enumerate(range(0, s, kc)):
            b1 = min(s, b0 + kc)
            chunk = mid[b0:b1].clone()
            dist.reduce(chunk, dst=c % world)
            if rank == c % world:
                acc += g[b0:b1].T @ chunk.numpy()
        accT = torch.from_numpy(acc)
        dist.all_reduce(accT)
        ref = g.T @ full_mid
        err = np.linalg.norm(accT.numpy() - ref) / np.linalg.norm(ref)
        result_q.put((rank, bool(ok_mid), float(err)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [1001, 4096])
def test_row_sharded_combined_sketch_world2(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    seed = orc.derive_seed(42, 201)
    seed2 = orc.derive_seed(seed, 1)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, 17, 256, 64, seed, seed2, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_mid, err in res:
        assert ok_mid, f"rank {rank}: allreduced count partials differ from the full sketch"
        assert err <= 1e-12, f"rank {rank}: chunk-owner Gaussian stage rel err {err}"
