"""CPU tests of the multi-GPU slab plan (csrc/shard.hpp): the partition and
the two exchange schedules, executed between real processes over
torch.distributed (gloo, world sizes 2 and 3) with numpy stand-ins for the
device buffers.  Each rank starts from exactly what its GPU holds after its
own SYRK tiles (pair grids) or its own centred rows (covariance), runs the
schedule the library computes, and must end with its window bit-equal to the
one-device arrays.  The device side of the same schedule (pack / unpack
kernels, NCCL or in-process transport) is checked on the GPU against the
one-device covariance (tests/test_gpu_shard.py)."""
import os
import socket

import numpy as np
import pytest

TILE = 64  # GEMM row tile (gemm.cu BM)


def _api():
    from paper_1510_04439_b200 import api
    return api


def tile_sym(X):
    """The one-device pair grid: upper tiles (tile(s) <= tile(t)) as computed,
    the rest mirrored (gemm.cu symmetric mode)."""
    G = X.shape[0]
    ts = np.arange(G) // TILE
    upper = ts[:, None] <= ts[None, :]
    return np.where(upper, X, X.T)


@pytest.mark.parametrize("n1,rn,R,world", [(64, 16, 7, 2), (64, 16, 7, 3), (64, 16, 3, 8), (32, 32, 4, 4),
                                           (100, 1, 25, 3), (16, 64, 7, 8)])
def test_bounds_partition_and_balance(n1, rn, R, world):
    api = _api()
    b = api.shard_bounds(n1, rn, R, world)
    assert b[0] == 0 and b[-1] == n1 and all(x <= y for x, y in zip(b, b[1:]))
    unit = TILE // np.gcd(rn, TILE)
    assert all(x % unit == 0 or x == n1 for x in b)  # slab starts on GEMM tile rows
    w = np.array([n1 - x - 0.5 for x in range(n1)])
    loads = [w[b[r]:b[r + 1]].sum() for r in range(world)]
    units = -(-n1 // unit)
    if units >= 4 * world:  # enough units to balance: within one unit's weight of the ideal
        assert max(loads) - w.sum() / world <= unit * n1


def simulate_phase(n1, rn, R, world, phase, seed=0):
    """Single-process replay of a schedule; returns per-rank windows and truth."""
    api = _api()
    G = n1 * rn
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((G, G))
    truth = tile_sym(X) if phase == 0 else np.triu(X) + np.triu(X, 1).T
    b = api.shard_bounds(n1, rn, R, world)
    blocks = api.shard_blocks(n1, rn, R, world, phase)
    bufs, row0s = [], []
    for r in range(world):
        a_, b_ = b[r], b[r + 1]
        if phase == 0:
            ha, hb = max(0, a_ - R), min(n1, b_ + R)
            buf = np.full(((hb - ha) * rn, G), np.nan)
            buf[(a_ - ha) * rn:(b_ - ha) * rn, a_ * rn:] = truth[a_ * rn:b_ * rn, a_ * rn:]
            row0s.append(ha * rn)
        else:
            buf = np.full(((b_ - a_) * rn, G), np.nan)
            buf[:, a_ * rn:] = truth[a_ * rn:b_ * rn, a_ * rn:]
            row0s.append(a_ * rn)
        bufs.append(buf)
    before = [x.copy() for x in bufs]
    for (src, dst, r0, r1, c0, c1, tr) in blocks:
        if src == dst and not tr:
            continue
        sb, so = before[src], row0s[src]
        vals = sb[c0 - so:c1 - so, r0:r1].T if tr else sb[r0 - so:r1 - so, c0:c1]
        bufs[dst][r0 - row0s[dst]:r1 - row0s[dst], c0:c1] = vals
    return truth, b, bufs, row0s


@pytest.mark.parametrize("n1,rn,R,world", [(64, 16, 7, 2), (64, 16, 7, 3), (64, 16, 3, 5), (32, 32, 4, 4),
                                           (16, 64, 7, 8)])
@pytest.mark.parametrize("phase", [0, 1])
def test_schedule_completes_every_window(n1, rn, R, world, phase):
    truth, b, bufs, row0s = simulate_phase(n1, rn, R, world, phase)
    for r in range(world):
        a_, b_ = b[r], b[r + 1]
        if a_ == b_:
            continue
        if phase == 0:
            ha, hb = max(0, a_ - R), min(n1, b_ + R)
            win = bufs[r][:, ha * rn:]
            ref = truth[ha * rn:hb * rn, ha * rn:]
        else:
            win, ref = bufs[r], truth[a_ * rn:b_ * rn]
        assert np.array_equal(win, ref), (r, phase)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_rank(rank, world, port, n1, rn, R, phase, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        api = _api()
        G = n1 * rn
        X = np.random.default_rng(7).standard_normal((G, G))  # same on every rank
        truth = tile_sym(X) if phase == 0 else np.triu(X) + np.triu(X, 1).T
        b = api.shard_bounds(n1, rn, R, world)
        a_, b_ = b[rank], b[rank + 1]
        if phase == 0:
            ha, hb = max(0, a_ - R), min(n1, b_ + R)
            row0 = ha * rn
            buf = np.full(((hb - ha) * rn, G), np.nan)
            buf[(a_ - ha) * rn:(b_ - ha) * rn, a_ * rn:] = truth[a_ * rn:b_ * rn, a_ * rn:]
        else:
            row0 = a_ * rn
            buf = np.full(((b_ - a_) * rn, G), np.nan)
            buf[:, a_ * rn:] = truth[a_ * rn:b_ * rn, a_ * rn:]
        blocks = api.shard_blocks(n1, rn, R, world, phase)
        # pack per destination (blocks in schedule order), like shard.cu
        out, inc, local = {}, {}, []
        for blk in blocks:
            src, dst, r0, r1, c0, c1, tr = (int(x) for x in blk)
            if src == rank:
                v = buf[c0 - row0:c1 - row0, r0:r1].T if tr else buf[r0 - row0:r1 - row0, c0:c1]
                if dst == rank:
                    if tr:
                        local.append((blk, v.copy()))
                else:
                    out.setdefault(dst, []).append(np.ascontiguousarray(v).ravel())
            if dst == rank and src != rank:
                inc.setdefault(src, []).append(blk)
        reqs = []
        for dst in sorted(out):
            reqs.append(dist.isend(torch.from_numpy(np.concatenate(out[dst])), dst))
        for src in sorted(inc):
            n = sum(int((k[3] - k[2]) * (k[5] - k[4])) for k in inc[src])
            t = torch.empty(n, dtype=torch.float64)
            dist.recv(t, src)
            msg, o = t.numpy(), 0
            for (s_, d_, r0, r1, c0, c1, tr) in (tuple(int(x) for x in k) for k in inc[src]):
                m = (r1 - r0) * (c1 - c0)
                buf[r0 - row0:r1 - row0, c0:c1] = msg[o:o + m].reshape(r1 - r0, c1 - c0)
                o += m
        for r in reqs:
            r.wait()
        for blk, v in local:
            src, dst, r0, r1, c0, c1, tr = (int(x) for x in blk)
            buf[r0 - row0:r1 - row0, c0:c1] = v
        if a_ < b_:
            if phase == 0:
                ok = np.array_equal(buf[:, ha * rn:], truth[ha * rn:hb * rn, ha * rn:])
            else:
                ok = np.array_equal(buf, truth[a_ * rn:b_ * rn])
        else:
            ok = True
        q.put((rank, bool(ok)))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("phase", [0, 1])
def test_schedule_over_gloo(world, phase):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_rank, args=(r, world, port, 64, 16, 7, phase, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    res = dict(q.get(timeout=5) for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    assert all(res[r] for r in range(world)), res
