"""World-size-2 CPU (gloo) tests of the row-sharded decompositions behind the
SRHT and rSVD paths; the arithmetic runs in the CPU oracle, the
collectives are real torch.distributed gloo collectives across processes.

* SRHT (csrc/srht.cu srht_rows_sharded): each rank cuts its rows into aligned
  power-of-two blocks (the last rank owns the zero padding), transforms each
  block with H_{2^b}, gathers the sampled outputs t at t mod 2^b with the
  Kronecker sign (-1)^popcount(offset & t), and one allreduce sums the ranks.
* rSVD (csrc/api_linalg.cpp KsvdWork::orth, sharded): CholeskyQR2 with an
  allreduced Gram, TSQR fallback from allgathered R factors, sign rule decided
  on the global row order (first rank with a decisive entry wins), and the
  allreduced A'Q / B' products.
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


def _blocks(row_off, n_local, n_total):
    """Aligned power-of-two blocks (offset, size, present) of srht_rows_sharded."""
    big_n = orc.next_pow2(n_total)
    end = row_off + n_local
    limit = big_n if end == n_total else end
    cur, out = row_off, []
    while cur < end:
        b = big_n if cur == 0 else (cur & -cur)
        while cur + b > limit:
            b >>= 1
        out.append((cur, b, min(b, end - cur)))
        cur += b
    return out


def _allreduce(x):
    t = torch.from_numpy(np.ascontiguousarray(x))
    dist.all_reduce(t)
    return t.numpy()


def _sign_fix_global(q_local, rank, world):
    """fix_column_signs_sharded: per-rank lead signs, allgathered, first decisive rank wins."""
    cols = q_local.shape[1]
    lead = np.zeros(cols)
    for j in range(cols):
        nz = np.nonzero(np.abs(q_local[:, j]) > 1e-12)[0]
        if nz.size:
            lead[j] = -1.0 if q_local[nz[0], j] < 0 else 1.0
    allv = np.zeros((world, cols))
    allv[rank] = lead
    allv = _allreduce(allv)
    flip = np.zeros(cols, dtype=bool)
    for j in range(cols):
        for r in range(world):
            if allv[r, j] != 0:
                flip[j] = allv[r, j] < 0
                break
    q_local[:, flip] *= -1
    return q_local


def _orth_sharded(y_local, rank, world, force_tsqr=False):
    cols = y_local.shape[1]
    if not force_tsqr:
        q = y_local.copy()
        ok = True
        for _ in range(2):
            g = _allreduce(q.T @ q)
            try:
                r = np.linalg.cholesky(g).T
            except np.linalg.LinAlgError:
                ok = False
                break
            q = q @ np.linalg.inv(r)
        if ok:
            return _sign_fix_global(q, rank, world)
    q_i, r_i = orc.thin_qr(y_local)
    stack = np.zeros((world, cols, cols))
    stack[rank] = r_i
    stack = _allreduce(stack).reshape(world * cols, cols)
    qs, _ = orc.thin_qr(stack)
    q = q_i @ qs[rank * cols:(rank + 1) * cols]
    return _sign_fix_global(q, rank, world)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {}
    try:
        # ---- SRHT ------------------------------------------------------------
        for n in (1000, 4096, 5001):
            rng = np.random.default_rng(n)
            d, s, seed = 5, 64, 77
            m = rng.standard_normal((n, d))
            signs, idx = orc.srht_operator(n, s, seed)
            r0, r1 = rn.shard_rows(n, world, rank)
            acc = np.zeros((s, d))
            for off, b, present in _blocks(r0, r1 - r0, n):
                x = np.zeros((b, d))
                x[:present] = m[off:off + present] * signs[off:off + present, None]
                hx = np.stack([orc.fwht(x[:, c]) for c in range(d)], axis=1)
                sgn = np.array([-1.0 if bin(off & int(t)).count("1") & 1 else 1.0 for t in idx])
                acc += sgn[:, None] * hx[np.asarray(idx) & (b - 1)] / np.sqrt(s)
            acc = _allreduce(acc)
            ref = orc.srht_rows(m, s, seed)
            out[f"srht{n}"] = float(np.linalg.norm(acc - ref) / np.linalg.norm(ref))
        # ---- rSVD with q = 1 power iteration ------------------------------------
        m_, n_, k, s = 600, 120, 6, 12
        rng = np.random.default_rng(5)
        u, _ = np.linalg.qr(rng.standard_normal((m_, n_)))
        v, _ = np.linalg.qr(rng.standard_normal((n_, n_)))
        a = (u * np.exp(-np.arange(1, n_ + 1) / 10.0)) @ v.T
        r0, r1 = rn.shard_rows(m_, world, rank)
        omega = orc.gaussian_matrix(n_, s, 31) / np.sqrt(s)
        for mode in ("cholqr", "tsqr"):
            tsqr = mode == "tsqr"
            y = a[r0:r1] @ omega
            qy = _orth_sharded(y, rank, world, tsqr)
            z = _allreduce(a[r0:r1].T @ qy)
            z, _ = orc.thin_qr(z)
            y = a[r0:r1] @ z
            qy = _orth_sharded(y, rank, world, tsqr)
            b = _allreduce(qy.T @ a[r0:r1])
            ub, sv, _ = orc.truncated_svd(b, k)
            u_loc = qy @ ub
            uo, so, _, _ = orc.prototype_ksvd(a, k, s, 31, q=1)
            out[f"sv_{mode}"] = float(np.max(np.abs(sv - so) / so))
            out[f"u_{mode}"] = float(np.max(np.abs(u_loc - uo[r0:r1])))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_sharded_srht_and_rsvd_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, out in res:
        for key, val in out.items():
            tol = 1e-12 if key.startswith("srht") else (1e-10 if key.startswith("sv") else 1e-8)
            assert val <= tol, f"rank {rank}: {key} = {val}"
