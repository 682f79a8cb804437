"""Full-size parity at every BASELINE.json config shape.

Each case runs the product path exactly as bench.py does — K1 on the whole
[M x K] activation (FP16 input for the linears that consume a gathered FP16
activation in the decoder layer, FP32 otherwise), then the fused K5 the planner
picks for M — and compares sampled rows with the reference's own
``dgq_forward`` (oracle/_ref = /root/reference/proj/src built unmodified):

* INT8 activation codes and row scales: bit-exact;
* INT32 accumulators: bit-exact (the oracle's W_s8 times its codes, exact in f64);
* FP32 output: bit-exact; FP16 output: == fp16_round(FP32 reference) bit-exact,
  which implies the stated tolerance |y16 - y| <= 2^-11 |y| + 2^-24.

Rows are independent in dgq_forward (proj/src/kernel.cpp:144-153), so a row
subset of the full-size layer is a complete check of those rows.  The rows
include the first/last rows of token tiles (128/256/512-row tiles) and the
last row, and every sampled row spans every weight tile, so tiles whose k-range
is split across CTA pairs by stream-K are covered.  Layers are random (not
periodic), so a kernel reading the wrong weight tile cannot pass.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2310_04836_b200 as dgq

pytestmark = pytest.mark.gpu

G = 128


def fast_layer(h: int, o: int, g: int, seed: int) -> oracle.Layer:
    """A valid random layer (SURVEY.md §8d flavour A: S2 in [1,127], ZP in [0,15],
    codes uniform in clip_interval(S2, ZP)) drawn with numpy's PCG64 — the
    SplitMix64 generator costs minutes at 205 M codes."""
    rng = np.random.default_rng(seed)
    ng = h // g
    s2 = rng.integers(1, 128, (ng, o), dtype=np.int16)
    zp = rng.integers(0, 16, (ng, o), dtype=np.int16)
    q = 127 // s2
    lo = np.maximum(0, zp - q).astype(np.uint8)
    span = (np.minimum(15, zp + q) - lo + 1).astype(np.uint8)
    codes = rng.integers(0, 1 << 16, (h, o), dtype=np.uint16)
    codes %= np.repeat(span, g, axis=0)
    codes = codes.astype(np.uint8) + np.repeat(lo, g, axis=0)
    s1c = 1.0 / (32.0 * h ** 0.5)  # bench.py's scale: outputs stay in FP16 range
    s1 = rng.uniform(0.5 * s1c, 1.5 * s1c, o).astype(np.float32)
    k = dgq.synth.smooth_k(h)  # the reference's smoothing recipe: k == 1 off the top 0.5 % channels
    return oracle.Layer(h=h, o=o, g=g, codes=oracle.pack_u4(codes), s2=s2.astype(np.int8).ravel(),
                        zp=oracle.pack_u4(zp.astype(np.uint8)), s1=s1, k=k, act_scale=0.0, mode=1)


def column_slice(L: oracle.Layer, c0: int, c1: int) -> oracle.Layer:
    """Columns [c0, c1) of a layer (c0, c1 even: nibble-aligned), the oracle-side
    view of a column-parallel shard."""
    ng = L.h // L.g
    return oracle.Layer(h=L.h, o=c1 - c0, g=L.g,
                        codes=np.ascontiguousarray(L.codes.reshape(L.h, L.o // 2)[:, c0 // 2:c1 // 2]).ravel(),
                        s2=np.ascontiguousarray(L.s2.reshape(ng, L.o)[:, c0:c1]).ravel(),
                        zp=np.ascontiguousarray(L.zp.reshape(ng, L.o // 2)[:, c0 // 2:c1 // 2]).ravel(),
                        s1=L.s1[c0:c1].copy(), k=L.k, act_scale=L.act_scale, mode=L.mode)


def to_dgq(L: oracle.Layer) -> dgq.DgqLayer:
    return dgq.DgqLayer(h=L.h, o=L.o, g=L.g, codes=L.codes, s2=L.s2.reshape(L.h // L.g, L.o), zp=L.zp, s1=L.s1,
                        k=L.k, act_scale=L.act_scale, mode=L.mode)


def sample_rows(M: int, seed: int) -> np.ndarray:
    fixed = [0, 1, 127, 128, 255, 256, 511, 512, M // 2, M - 257, M - 129, M - 1]
    rnd = np.random.default_rng(seed).integers(0, M, 2).tolist()
    return np.array(sorted({r for r in fixed + rnd if 0 <= r < M}))


def activations(M: int, K: int, seed: int, f16: bool) -> torch.Tensor:
    x = torch.from_numpy(dgq.synth.gen_synthetic(M, K, seed, 3, 50.0, 7))
    return x.half() if f16 else x


_layers: dict = {}


def layer_for(h: int, o: int, g: int, seed: int, c0: int = 0, c1: int | None = None):
    """(oracle layer of the shard, CudaLayer of the shard) — built once per session."""
    key = (h, o, g, seed, c0, c1)
    if key not in _layers:
        if len(_layers) >= 2:  # keep host/device memory bounded
            _layers.clear()
            torch.cuda.empty_cache()
        L = fast_layer(h, o, g, seed)
        c1 = c1 or o
        CL = dgq.CudaLayer(to_dgq(L), col_begin=c0, col_end=c1)
        _layers[key] = (column_slice(L, c0, c1) if (c0, c1) != (0, o) else L, CL)
    return _layers[key]


def check(ref, Lo: oracle.Layer, CL: dgq.CudaLayer, M: int, f16_in: bool, seed: int):
    x = activations(M, Lo.h, seed, f16_in)
    xd = x.cuda()
    codes, rs = CL.quantize_act(xd)
    y16 = CL.linear(codes, rs, out_dtype=torch.float16)           # the bench's launch
    y32, acc = CL.linear(codes, rs, out_dtype=torch.float32, want_acc=True)
    torch.cuda.synchronize()
    rows = sample_rows(M, seed)
    xr = x[rows].float().numpy()
    out, w, q, rsr, _ = ref.dgq_forward(xr, Lo, None, 0)
    got_codes = codes[rows][:, :Lo.h].cpu().numpy()
    assert np.array_equal(got_codes, q), "activation codes"
    assert not codes[:, Lo.h:].any(), "pad columns must be zero"
    assert np.array_equal(rs[rows].cpu().numpy().view(np.uint32), rsr.view(np.uint32)), "row scales"
    acc_ref = (q.astype(np.float64) @ w.astype(np.float64)).astype(np.int64)  # exact: |partial sums| < 2^31
    assert np.array_equal(acc[rows].cpu().numpy().astype(np.int64), acc_ref), "int32 accumulators"
    assert np.array_equal(y32[rows].cpu().numpy().view(np.uint32), out.view(np.uint32)), "FP32 output"
    ref16 = oracle.fp16_round_np(out).astype(np.float16)
    got16 = y16[rows].cpu().numpy()
    assert np.array_equal(got16.view(np.uint16), ref16.view(np.uint16)), "FP16 output"
    d = np.abs(got16.astype(np.float64) - out.astype(np.float64))
    assert (d <= np.abs(out) * 2.0 ** -11 + 2.0 ** -24 + 1e-30).all()
    return CL.plan(M)


# C3: OPT-30B decoder-layer linears at seq 512 / 1024 / 2048 (bench.py's step).
# q reads the FP32 layer input; out / fc1 / fc2 read a gathered FP16 activation.
OPT30B = [("q", 7168, 7168, False), ("out", 7168, 7168, True), ("fc1", 7168, 28672, True),
          ("fc2", 28672, 7168, True)]


@pytest.mark.parametrize("name,K,N,f16", OPT30B, ids=[c[0] for c in OPT30B])
def test_opt30b_prefill_full_size(cuda, ref, name, K, N, f16):
    Lo, CL = layer_for(K, N, G, seed=K + N)
    for M in (512, 1024, 2048):
        plan = check(ref, Lo, CL, M, f16, seed=M + K)
        assert plan["token_tile"] >= 256, plan  # the CTA-pair kernel (K5p) at these sizes


@pytest.mark.parametrize("M", [1, 16, 32])
def test_opt30b_decode_full_size(cuda, ref, M):
    for K, N in ((7168, 7168), (7168, 28672), (28672, 7168)):
        Lo, CL = layer_for(K, N, G, seed=K + N)
        check(ref, Lo, CL, M, M > 1, seed=M + K)


# C2: LLaMA-7B layer GEMMs (qkv / o 4096^2, up / gate 4096 -> 11008, down 11008 -> 4096)
LLAMA7B = [("qkv", 4096, 4096), ("up", 4096, 11008), ("down", 11008, 4096)]


@pytest.mark.parametrize("name,K,N", LLAMA7B, ids=[c[0] for c in LLAMA7B])
def test_llama7b_full_size(cuda, ref, name, K, N):
    Lo, CL = layer_for(K, N, G, seed=K * 3 + N)
    for M in (2048, 1):
        check(ref, Lo, CL, M, name == "down", seed=M + N)


# C4: LLaMA-65B FFN on one 8-way column shard (N/8 = 2752 / 1024), decode batch 1-64
LLAMA65B = [("up", 8192, 22016, 5), ("down", 22016, 8192, 2)]


@pytest.mark.parametrize("name,K,N,rank", LLAMA65B, ids=[c[0] for c in LLAMA65B])
def test_llama65b_shard_decode(cuda, ref, name, K, N, rank):
    shard = N // 8
    Lo, CL = layer_for(K, N, G, seed=K + 2 * N, c0=rank * shard, c1=(rank + 1) * shard)
    assert CL.o == shard
    for M in (1, 2, 4, 8, 16, 32, 64):
        check(ref, Lo, CL, M, name == "down", seed=M)


# C1 / C5: M in {1, 16}, K = N = 4096, g in {64, 128}; plus the M sweep's ragged points
@pytest.mark.parametrize("g", [64, 128])
def test_c1_square_4096(cuda, ref, g):
    Lo, CL = layer_for(4096, 4096, g, seed=g)
    for M in (1, 16, 3, 48, 100, 333, 4096):
        check(ref, Lo, CL, M, False, seed=M * g)
