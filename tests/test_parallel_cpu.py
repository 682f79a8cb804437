"""Multi-process host logic of the column-parallel path, on CPU with gloo
(world_size 2 and 4): each rank computes its column shard with the CPU oracle
from `shard_layer`, the shards are all-gathered in the [p][M][N/p] layout, and
the reassembled output must equal the unsharded layer bit-for-bit (the same
property the GPU path relies on)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2310_04836_b200 as dgq
from paper_2310_04836_b200 import parallel


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _to_oracle(L: dgq.DgqLayer) -> oracle.Layer:
    codes, s2, zp, s1, k = L.arrays()
    return oracle.Layer(h=L.h, o=L.o, g=L.g, codes=codes, s2=s2, zp=zp, s1=s1, k=k, act_scale=L.act_scale,
                        mode=L.mode)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        P = oracle.port()
        L = dgq.random_layer(256, 96, 64, seed=5)
        X = P.gen_synthetic(12, 256, 9, 3, 50.0, 7)
        S = parallel.shard_layer(L, rank, world)
        out, *_ = P.dgq_forward(X, _to_oracle(S))
        local = torch.from_numpy(out)
        g = torch.empty(world * 12, S.o, dtype=torch.float32)
        dist.all_gather_into_tensor(g, local)
        full = parallel.gathered_to_full(g.view(world, 12, S.o).numpy())
        if rank == 0:
            ref, *_ = P.dgq_forward(X, _to_oracle(L))
            q.put(bool(np.array_equal(full.view(np.uint32), ref.view(np.uint32))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_column_parallel_gloo_matches_unsharded(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert q.get(timeout=5) is True


def test_shard_range_and_errors():
    assert parallel.shard_range(28672, 3, 8) == (10752, 14336)
    with pytest.raises(ValueError):
        parallel.shard_range(30, 4, 4)  # 30 / 4 is not integral
    with pytest.raises(ValueError):
        parallel.shard_range(12, 0, 4)  # width 3 is odd


def test_shard_layer_concatenates_back():
    L = dgq.random_layer(64, 48, 16, seed=2)
    parts = [parallel.shard_layer(L, r, 3) for r in range(3)]
    P = oracle.port()
    full = P.dequantize_to_s8(_to_oracle(L))
    got = np.concatenate([P.dequantize_to_s8(_to_oracle(s)) for s in parts], axis=1)
    assert np.array_equal(full, got)
    assert np.array_equal(np.concatenate([s.s1 for s in parts]), L.s1)


def test_gathered_layout_roundtrip():
    g = np.arange(2 * 3 * 4).reshape(2, 3, 4)
    full = parallel.gathered_to_full(g)
    assert full.shape == (3, 8)
    assert np.array_equal(full[:, 4:], g[1])
