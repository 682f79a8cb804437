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


class _OracleShard:
    """A CPU stand-in for a rank's CudaLayer shard (same quantize_act / linear
    interface), computing with the pinned C restatement: lets ColumnParallelLinear
    itself — sharding, the gathered [p][M][N/p] layout, the all-gather and the
    next layer's K1 on the gathered input — run over gloo without a GPU."""

    def __init__(self, L, c0, c1):
        self.P = oracle.port()
        self.S = _to_oracle(parallel.shard_layer(L, c0 // (c1 - c0), L.o // (c1 - c0)))
        self.w = self.P.dequantize_to_s8(self.S)

    def quantize_act(self, x, codes=None, rs=None):
        if x.dim() == 3:  # the gathered [p][M][N/p] activation, read in place on the GPU
            x = parallel.gathered_to_full(x)
        q, r = self.P.quantize_activations(x.float().numpy(), self.S.k, self.S.mode, self.S.act_scale)
        return torch.from_numpy(q), torch.from_numpy(r)

    def linear(self, codes, rs, bias=None, out=None, out_dtype=torch.float16):
        acc, _ = self.P.int8_gemm(codes.numpy(), self.w)
        y = self.P.epilogue(acc, rs.numpy(), self.S.s1)
        if out_dtype == torch.float16:
            return torch.from_numpy(oracle.fp16_round_np(y).astype(np.float16))
        return torch.from_numpy(y)

    def close(self):
        pass


def _chain_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        L1 = dgq.random_layer(256, 32 * world, 64, seed=11)
        L2 = dgq.random_layer(32 * world, 16 * world, 32, seed=12)
        X = oracle.port().gen_synthetic(10, 256, 5, 3, 50.0, 7)
        a = parallel.ColumnParallelLinear(L1, rank, world, shard_factory=_OracleShard)
        b = parallel.ColumnParallelLinear(L2, rank, world, shard_factory=_OracleShard)
        h1 = a(torch.from_numpy(X))           # [p][M][N1/p] FP16, all-gathered
        y = b(h1, gather=True, out_dtype=torch.float32)   # K1 on the gathered layout, then gather again
        if rank == 0:
            P = oracle.port()
            r1, *_ = P.dgq_forward(X, _to_oracle(L1))
            x2 = oracle.fp16_round_np(r1).astype(np.float16).astype(np.float32)
            r2, *_ = P.dgq_forward(x2, _to_oracle(L2))
            full = parallel.gathered_to_full(y.numpy())
            q.put(bool(np.array_equal(full.view(np.uint32), r2.view(np.uint32))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_column_parallel_linear_chain_over_gloo(world):
    # two chained column-parallel linears through ColumnParallelLinear itself
    # (FP16 all-gather between them, the next K1 reading the gathered layout):
    # the reassembled output equals the unsharded computation bit for bit
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_chain_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
        assert p.exitcode == 0
    assert q.get(timeout=5) is True
