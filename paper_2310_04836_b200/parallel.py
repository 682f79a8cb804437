"""Column-parallel (N-sharded) DGQ linears across the GPUs of one node
(SURVEY.md §8e).

Rank r of p owns output channels [r*N/p, (r+1)*N/p): its codes / S2 / ZP
columns and s1 slice; k, act_scale and the activations are replicated, and
K1 runs redundantly on every rank (deterministic, so every rank holds
bit-identical codes and row scales — no broadcast).  Each output column is
computed exactly as on one GPU, so integer and FP32 results are bit-identical
to the unsharded layer.  The only exchange is an NCCL all-gather of the FP16
output where the consumer needs the full activation; the gathered buffer is
kept in its natural [p][M][N/p] layout and the next layer's K1 reads it in
place (dgq_quantize_act_f16 with seg_cols = N/p), so no permute pass exists.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .api import CudaLayer, DgqLayer


def shard_range(o: int, rank: int, world: int):
    """Columns of rank `rank`: equal, even-width shards (packed 4-bit storage)."""
    if o % world or (o // world) % 2:
        raise ValueError(f"output width {o} does not split into {world} even shards")
    w = o // world
    return rank * w, (rank + 1) * w


def shard_layer(layer: DgqLayer, rank: int, world: int) -> DgqLayer:
    """Host-side column shard in the reference layout (what dgq_layer_create's
    col_begin/col_end keeps on the device)."""
    c0, c1 = shard_range(layer.o, rank, world)
    codes, s2, zp, s1, k = layer.arrays()
    ng = layer.n_g
    w = c1 - c0
    codes2 = codes.reshape(layer.h, layer.o // 2)[:, c0 // 2:c1 // 2].copy()
    s22 = s2.reshape(ng, layer.o)[:, c0:c1].copy()
    zp2 = zp.reshape(ng, layer.o // 2)[:, c0 // 2:c1 // 2].copy()
    return DgqLayer(h=layer.h, o=w, g=layer.g, codes=codes2.ravel(), s2=s22, zp=zp2.ravel(), s1=s1[c0:c1].copy(),
                    k=k.copy(), act_scale=layer.act_scale, mode=layer.mode)


def gathered_to_full(g):
    """[p, M, N/p] (all-gather layout) -> [M, N]."""
    if isinstance(g, torch.Tensor):
        p, M, w = g.shape
        return g.permute(1, 0, 2).reshape(M, p * w)
    p, M, w = g.shape
    return np.ascontiguousarray(np.transpose(g, (1, 0, 2)).reshape(M, p * w))


class ColumnParallelLinear:
    """One DGQ linear, column-sharded over the ranks of `group`.

    `shard_factory(layer, c0, c1)` builds the rank's shard (default: a CudaLayer
    holding columns [c0, c1) on `device`); anything with the same
    quantize_act / linear interface works, which is how the multi-process CPU
    tests run this class over gloo with an oracle-backed shard."""

    def __init__(self, layer: DgqLayer, rank: int = 0, world: int = 1, device=None, group=None,
                 validate: bool = True, shard_factory=None):
        self.rank, self.world, self.group = rank, world, group
        self.o_full = layer.o
        self.c0, self.c1 = shard_range(layer.o, rank, world)
        if shard_factory is None:
            self.layer = CudaLayer(layer, device=device, col_begin=self.c0, col_end=self.c1, validate=validate)
        else:
            self.layer = shard_factory(layer, self.c0, self.c1)
        self.h = layer.h
        self.shard = self.c1 - self.c0

    def quantize(self, x, codes=None, rs=None):
        """K1 on the full input: float32/float16 [M, h] or a gathered float16 [p, M, h/p]."""
        return self.layer.quantize_act(x, codes, rs)

    def linear(self, codes, rs, out=None, out_dtype=torch.float16, bias=None):
        return self.layer.linear(codes, rs, bias=bias, out=out, out_dtype=out_dtype)

    def gather(self, local: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """NCCL all-gather of the [M, N/p] shard -> [p, M, N/p]."""
        M = local.shape[0]
        if self.world == 1:
            return local.unsqueeze(0)
        if out is None:
            out = torch.empty(self.world, M, self.shard, dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(out.view(self.world * M, self.shard), local.contiguous(), group=self.group)
        return out

    def __call__(self, x, gather: bool = True, out_dtype=torch.float16):
        codes, rs = self.quantize(x)
        y = self.linear(codes, rs, out_dtype=out_dtype)
        return self.gather(y) if gather else y

    def close(self):
        self.layer.close()


class DgqComm:
    """The C-ABI communicator (dgq_comm_create over NCCL) for callers of
    dgq_linear_allgather: rank 0 draws the unique id, torch.distributed (any
    backend) broadcasts it; world 1 needs no process group."""

    def __init__(self, rank: int = 0, world: int = 1, device=None, group=None):
        import ctypes as C

        from ._lib import check, lib

        uid = (C.c_uint8 * 128)()
        if rank == 0:
            check(lib().dgq_comm_unique_id(uid))
        if world > 1:
            obj = [bytes(uid)]
            dist.broadcast_object_list(obj, src=0, group=group)
            uid = (C.c_uint8 * 128).from_buffer_copy(obj[0])
        self.device = torch.cuda.current_device() if device is None else torch.device(device).index
        self._h = C.c_void_p()
        check(lib().dgq_comm_create(world, rank, uid, self.device, C.byref(self._h)))
        self.world = world

    def linear_allgather(self, lin: "ColumnParallelLinear", codes: torch.Tensor, rs: torch.Tensor,
                         out_dtype=torch.float16, bias: torch.Tensor | None = None):
        """dgq_linear_allgather: this rank's shard, then the [p][M][N/p] all-gather."""
        import ctypes as C

        from ._lib import OUT_F16, OUT_F32, check, lib

        M = codes.shape[0]
        local = torch.empty(M, lin.shard, dtype=out_dtype, device=codes.device)
        full = torch.empty(self.world, M, lin.shard, dtype=out_dtype, device=codes.device)
        check(lib().dgq_linear_allgather(lin.layer.handle, C.c_void_p(codes.data_ptr()), codes.stride(0),
                                         C.c_void_p(rs.data_ptr()), M,
                                         None if bias is None else C.c_void_p(bias.data_ptr()),
                                         OUT_F16 if out_dtype == torch.float16 else OUT_F32,
                                         C.c_void_p(local.data_ptr()), C.c_void_p(full.data_ptr()), self._h,
                                         C.c_void_p(torch.cuda.current_stream(codes.device).cuda_stream)))
        return full

    def close(self):
        from ._lib import lib

        if self._h and self._h.value:
            lib().dgq_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
