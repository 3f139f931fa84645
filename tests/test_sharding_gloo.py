"""N>1 host path on CPU (gloo, world_size 2): requests shard round-robin with no data-path
collective, each rank plans ONE batched device pass over its shard, and the per-request
results of the batched plan equal the single-request plans (the reference's rows and
computed_per_layer, plans.py:104-114 / engine.py:161-163)."""
import os
import socket
from types import SimpleNamespace

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_12977_b200.layout import build_layout
from paper_2512_12977_b200.sharding import gather_metadata, head_split, shard_indices
from test_host_cpu import _spec

L, T = 4, 64


def _requests(n):
    rng = np.random.default_rng(5)
    out = []
    for i in range(n):
        nimg = int(rng.integers(1, 4))
        r = [0.3, 0.1, 0.05, 0.0][int(rng.integers(0, 4))]
        ratios = tuple(sorted([r, r / 2 if r != 0.05 else 0.05, 0.0, 0.0], reverse=True))
        ratios = tuple(round(round(x / 0.002) * 0.002, 3) for x in ratios)
        out.append((int(rng.integers(0, 9)), nimg, int(rng.integers(0, 9)), ratios))
    return out


def _single(req):
    pre, nimg, suf, ratios = req
    _, _, spec = _spec(pre, T, nimg, suf, ratios)
    lay = build_layout([spec], L, heads=2)
    return lay.positions[0].tolist(), [int(c) for c in _counts(spec)]


def _counts(spec):
    return [len(spec.text_pos) + int(spec.keep[i].sum()) for i in range(L)]


def _worker(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        reqs = _requests(n)
        idx = shard_indices(n, rank, world)
        specs = [_spec(reqs[i][0], T, reqs[i][1], reqs[i][2], reqs[i][3])[2] for i in idx]
        lay = build_layout(specs, L, heads=2)          # one batched pass per rank
        results = [SimpleNamespace(positions=lay.positions[j],
                                   metrics=SimpleNamespace(computed_per_layer=_counts(specs[j])))
                   for j in range(len(idx))]
        # batched layout: layer i works on the concatenated computed rows of all requests
        for i in range(L):
            assert int(lay.c[i]) == sum(_counts(s)[i] for s in specs)
        got = gather_metadata(idx, results)
        if rank == 0:
            q.put(got)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_indices_partition():
    for n in (0, 1, 7, 64):
        for world in (1, 2, 3, 8):
            parts = [shard_indices(n, r, world) for r in range(world)]
            flat = sorted(i for p in parts for i in p)
            assert flat == list(range(n))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1


def test_head_split_uneven():
    assert [k for _, k in head_split(28, 8)] == [4, 4, 4, 4, 3, 3, 3, 3]
    assert head_split(28, 2) == [(0, 14), (14, 14)]
    with pytest.raises(ValueError):
        head_split(4, 8)


@pytest.mark.timeout(300)
def test_gloo_two_ranks_batched_shards_equal_single_requests():
    n = 9
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [g[0] for g in got] == list(range(n))
    reqs = _requests(n)
    for i, pos, counts in got:
        want_pos, want_counts = _single(reqs[i])
        assert pos == want_pos
        assert counts == want_counts
