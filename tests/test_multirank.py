"""World-size-2 (gloo, CPU) test of the multi-GPU host path.

On B200 the per-batch exchange runs over NCCL inside libomcg: an int64
all-reduce of tallies/k-eff accumulators, an all-gather of per-rank fission
bank sizes, and grouped send/recv of the canonical bank slices given by
omcg_bank_exchange_plan. Here the same plan (the product's C function) drives
the same collectives over gloo and the resampled next-batch source on every
rank must equal the single-rank result exactly.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

SITE = 5  # x, y, z, E (f64 bits) + key, as int64 words


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _global_bank(N, seed):
    """A canonical global fission bank: sites ordered by (history, progeny)."""
    rng = np.random.default_rng(seed)
    per = rng.poisson(1.0, N)  # sites per history
    hist = np.repeat(np.arange(N), per)
    prog = np.concatenate([np.arange(k) for k in per]) if per.sum() else np.zeros(0, int)
    sites = np.zeros((len(hist), SITE), np.int64)
    sites[:, :4] = rng.integers(0, 2**62, (len(hist), 4))
    sites[:, 4] = (hist << 24) | prog
    return sites, hist


def _resample(bank, S, off, N, lo, n):
    gi = np.arange(lo, lo + n, dtype=np.uint64)
    idx = (gi * np.uint64(S) + np.uint64(off)) // np.uint64(N)
    return idx.astype(np.int64)


def _worker(rank, world, port, N, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2402_09222_b200 as P

    bank, hist = _global_bank(N, seed)
    lo, hi = N * rank // world, N * (rank + 1) // world
    mine = bank[(hist >= lo) & (hist < hi)]  # this rank's canonical slice
    # all-gather bank sizes
    sz = torch.tensor([len(mine)], dtype=torch.int64)
    all_sz = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(all_sz, sz)
    S_all = np.array([int(t) for t in all_sz], np.uint64)
    S = int(S_all.sum())
    off = (S * 7919) % S
    plan = P.bank_exchange_plan(S_all, N, off, rank)
    W = world
    need_first, need_count = int(plan[4 * W]), int(plan[4 * W + 1])
    recv = np.zeros((need_count, SITE), np.int64)
    reqs = []
    for r in range(W):
        sf, sc, rf, rc = (int(plan[k * W + r]) for k in range(4))
        if r == rank:
            recv[rf:rf + rc] = mine[sf:sf + sc]
            continue
        if sc:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(mine[sf:sf + sc])), dst=r))
        if rc:
            buf = torch.zeros((rc, SITE), dtype=torch.int64)
            reqs.append((dist.irecv(buf, src=r), buf, rf, rc))
    for item in reqs:
        if isinstance(item, tuple):
            item[0].wait()
            recv[item[2]:item[2] + item[3]] = item[1].numpy()
        else:
            item.wait()
    idx = _resample(None, S, off, N, lo, hi - lo)
    source = recv[idx - need_first]
    # integer tally reduction is exact regardless of rank count
    tally = torch.from_numpy(np.random.default_rng(rank).integers(0, 2**40, 64))
    dist.all_reduce(tally)
    q.put((rank, source, tally.numpy(), S, off))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_bank_redistribution_matches_single_rank(world):
    N, seed = 5003, 11
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, N, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict()
    for _ in range(world):
        rank, source, tally, S, off = q.get(timeout=120)
        out[rank] = (source, tally, S, off)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    bank, _ = _global_bank(N, seed)
    S, off = out[0][2], out[0][3]
    full = bank[_resample(None, S, off, N, 0, N)]
    got = np.concatenate([out[r][0] for r in range(world)])
    assert np.array_equal(got, full)
    want_tally = sum(np.random.default_rng(r).integers(0, 2**40, 64) for r in range(world))
    for r in range(world):
        assert np.array_equal(out[r][1], want_tally)
