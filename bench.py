#!/usr/bin/env python
"""DGQ A8W4 benchmark (driver contract).

One step = one OPT-30B decoder layer's six DGQ linears at seq M = 2048
(q, k, v, out 7168x7168; fc1 7168x28672; fc2 28672x7168; g = 128, FP16 out)
plus the four K1 activation quantisations (one per distinct input: q/k/v
share theirs, and run as ONE fused-linear launch over their three weight sets,
dgq_linear_multi — four K5 launches per step).  Weights are column-sharded over the N ranks; the out / fc1 /
fc2 outputs and the attention stand-in (the q output) are NCCL all-gathered
and the next K1 reads the gathered [p][M][N/p] buffer in place.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

value = whole-job INT8 TOPS of the step (2*M*sum(K*N) / max-over-ranks time),
inputs resident in HBM, L2 flushed (256 MiB write) between timed steps.
e2e   = the same step through the public API with the f32 input copied from
pinned host memory and the rank's fc2 output shard copied back, every step.
--impl reference times the reference's own CPU implementation
(oracle/_ref = /root/reference/proj/src built unmodified) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "A8W4 GEMM TOPS & HBM GB/s (roofline %); OPT-30B layer ms @ seq 512–2048"
UNIT = "TOPS"
OPT30B = [("q", 7168, 7168), ("k", 7168, 7168), ("v", 7168, 7168), ("out", 7168, 7168), ("fc1", 7168, 28672),
          ("fc2", 28672, 7168)]
GROUP = 128
SEQ = 2048
# The CPU arms (--impl reference and our cpu_baseline) run the SAME step shape —
# the six OPT-30B decoder-layer linears at seq 2048, through the reference's own
# dgq_forward per linear (act quant + per-call weight dequant + int8 GEMM +
# epilogue) — bounded by restricting every linear to its first CPU_COLS output
# channels: M and K (and so the act-quant and GEMM shapes per column) are the
# headline's; only N shrinks.
CPU_COLS = 128
CPU_SAMPLE_DESC = (f"OPT-30B decoder-layer linears at seq 2048 (q,k,v,out 7168->{CPU_COLS}, fc1 7168->{CPU_COLS}, "
                   f"fc2 28672->{CPU_COLS}: each linear's first {CPU_COLS} output channels), one dgq_forward per "
                   f"linear incl. its per-call act quant and weight dequant, g=128, M=2048")


def layer_ops(M: int) -> float:
    return 2.0 * M * sum(k * n for _, k, n in OPT30B)


def layer_weight_bytes(world: int = 1) -> float:
    """Algorithmic HBM bytes of the weights per step per rank (codes + S2 + ZP + s1)."""
    b = 0.0
    for _, k, n in OPT30B:
        ns = n / world
        b += k * ns / 2 + (k / GROUP) * ns * 1.5 + 4 * ns
    return b


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        sm = [float(r[1]) for r in rows if len(r) > 2 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) > 2 and r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            for i, n in enumerate(names):
                if len(r) > 5 + i and "Active" in r[5 + i] and "Not" not in r[5 + i]:
                    reasons.add(n)
        busy = [s for s in sm if mx and s > 0.3 * max(mx)] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(rows)}


# ----------------------------------------------------------------------------- reference arm
def _cpu_layer_sample():
    """(oracle layers, inputs) of the bounded CPU step: every OPT-30B linear cut
    to its first CPU_COLS output channels, inputs at seq 2048."""
    from paper_2310_04836_b200 import synth

    Ls = [_oracle_layer(tiled_layer(K, CPU_COLS, seed=100 + i)) for i, (_, K, _) in enumerate(OPT30B)]
    xs = {K: synth.gen_synthetic(SEQ, K, 101 + K, 3, 50.0, 7) for K in sorted({k for _, k, _ in OPT30B})}
    ops = 2.0 * SEQ * CPU_COLS * sum(K for _, K, _ in OPT30B)
    return Ls, [xs[K] for _, K, _ in OPT30B], ops


def _cpu_step(be, Ls, Xs):
    for L, X in zip(Ls, Xs):
        be.dgq_forward(X, L, None, 0) if be.kind == "reference" else be.dgq_forward(X, L)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle

    be = oracle.best()
    Ls, Xs, ops = _cpu_layer_sample()
    cores = os.cpu_count() or 1
    for _ in range(args.warmup):
        _cpu_step(be, Ls, Xs)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        _cpu_step(be, Ls, Xs)
        ts.append(time.perf_counter() - t0)
    tot = sum(ts)
    val = ops * len(ts) / tot / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot / len(ts) * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int8 (i8 x i8 -> i32, fp32 epilogue)", "data": "synthetic",
        "config": {"workload": "OPT-30B decoder-layer linears, seq 2048 (column-bounded CPU sample)",
                   "sample": CPU_SAMPLE_DESC, "seq_len": SEQ, "group": GROUP},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": be.kind, "sample": CPU_SAMPLE_DESC},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _oracle_layer(L):
    import oracle

    codes, s2, zp, s1, k = L.arrays()
    return oracle.Layer(h=L.h, o=L.o, g=L.g, codes=codes, s2=s2, zp=zp, s1=s1, k=k, act_scale=L.act_scale,
                        mode=L.mode)


def cpu_baseline_sample():
    """Our arm's cpu_baseline: one bounded step of the reference arm's sample on the host cores."""
    import oracle

    be = oracle.best()
    Ls, Xs, ops = _cpu_layer_sample()
    t0 = time.perf_counter()
    _cpu_step(be, Ls, Xs)
    t = time.perf_counter() - t0
    return {"value": ops / t / 1e12, "unit": UNIT, "cores": os.cpu_count() or 1, "kind": be.kind,
            "sample": f"{CPU_SAMPLE_DESC}; one step ({t:.2f} s, threads = all host cores)"}


# ----------------------------------------------------------------------------- our arm
def tiled_layer(K: int, N: int, seed: int, k_vec=None, group: int = GROUP):
    """A valid random DGQ layer of width N built by tiling a 512-wide random
    block (values do not affect the data-independent kernels; building 205M
    random codes on the host per run would dominate the bench)."""
    import numpy as np

    from paper_2310_04836_b200 import DgqLayer, synth

    # s1 ~ 1 / (E|W_s8| sqrt(K)): outputs keep the scale of the inputs through the
    # chained linears (no normalisation between them here), as a real layer's
    # per-channel scales do; larger s1 overflow FP16 two linears down
    s1c = 1.0 / (32.0 * K ** 0.5)
    base = synth.random_layer(K, 512, group, seed=seed, s1_range=(0.5 * s1c, 1.5 * s1c))
    if k_vec is None:  # the reference's smoothing recipe: k == 1 off the top 0.5 % channels
        k_vec = synth.smooth_k(K)
    reps = -(-N // 512)
    codes = np.tile(base.codes.reshape(K, 256), (1, reps))[:, :N // 2]
    s2 = np.tile(base.s2.reshape(K // group, 512), (1, reps))[:, :N]
    zp = np.tile(base.zp.reshape(K // group, 256), (1, reps))[:, :N // 2]
    s1 = np.tile(base.s1, reps)[:N]
    return DgqLayer(h=K, o=N, g=group, codes=np.ascontiguousarray(codes).ravel(), s2=np.ascontiguousarray(s2),
                    zp=np.ascontiguousarray(zp).ravel(), s1=np.ascontiguousarray(s1), k=k_vec, act_scale=0.0, mode=1)


class OptLayer:
    """The six column-parallel linears of one OPT-30B decoder layer + buffers."""

    def __init__(self, rank, world, device, group, M_max):
        import torch

        from paper_2310_04836_b200.parallel import ColumnParallelLinear

        self.world, self.device, self.M_max = world, device, M_max
        qkv_k = None
        self.lin = {}
        self.host = {}  # host DgqLayers (reference layout) for the post-run self-check
        self.rank = rank
        for i, (name, K, N) in enumerate(OPT30B):
            L = tiled_layer(K, N, seed=100 + i, k_vec=qkv_k if name in ("k", "v") else None)
            if name == "q":
                qkv_k = L.k  # q/k/v share the input and its smoothing vector
            self.lin[name] = ColumnParallelLinear(L, rank, world, device, group)
            if name in ("fc1", "fc2"):
                self.host[name] = L
        f16 = torch.float16
        dev = device
        self.x = torch.empty(M_max, 7168, dtype=torch.float32, device=dev)
        self.codes = {n: torch.empty(M_max, self.lin[n].layer.k_pad, dtype=torch.int8, device=dev)
                      for n in ("q", "out", "fc1", "fc2")}
        self.rs = {n: torch.empty(M_max, dtype=torch.float32, device=dev) for n in ("q", "out", "fc1", "fc2")}
        self.y = {n: torch.empty(M_max, self.lin[n].shard, dtype=f16, device=dev) for n, _, _ in OPT30B}
        self.g = {n: torch.empty(world, M_max, self.lin[n].shard, dtype=f16, device=dev)
                  for n in ("q", "out", "fc1", "fc2")}
        self.k_events = []  # (start, end, ops) of the K5 launches while recording
        self.q_events = []  # (start, end, bytes) of the K1 launches while recording
        self.record = False

    def _k5(self, name, codes, rs, M, out=None):
        import torch

        lin = self.lin[name]
        if self.record:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
        lin.linear(codes[:M], rs[:M], out=self.y[name][:M] if out is None else out)
        if self.record:
            b.record()
            self.k_events.append((a, b, 2.0 * M * lin.h * lin.shard, name))

    def _k5_qkv(self, codes, rs, M):
        import torch

        from paper_2310_04836_b200 import linear_multi

        names = ("q", "k", "v")
        if self.record:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
        linear_multi([self.lin[n].layer for n in names], codes[:M], rs[:M], outs=[self.y[n][:M] for n in names])
        if self.record:
            b.record()
            ops = sum(2.0 * M * self.lin[n].h * self.lin[n].shard for n in names)
            self.k_events.append((a, b, ops, "qkv"))

    def _k1(self, name, x, M):
        import torch

        lin = self.lin[name]
        if self.record:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
        lin.quantize(x, self.codes[name][:M], self.rs[name][:M])
        if self.record:
            b.record()
            esz = x.element_size()
            self.q_events.append((a, b, (esz + 1) * M * lin.h + 4 * lin.h + 4 * M, name))

    def _gather(self, name, M, src=None):
        lin = self.lin[name]
        src = self.y[name][:M] if src is None else src
        if self.world == 1:
            return src.unsqueeze(0)
        if M == self.M_max:
            lin.gather(src, out=self.g[name])
            return self.g[name]
        import torch.distributed as dist

        buf = self.g[name].view(-1)[: self.world * M * lin.shard].view(self.world, M, lin.shard)
        dist.all_gather_into_tensor(buf.view(self.world * M, lin.shard), src.contiguous(), group=lin.group)
        return buf

    def step(self, M, x=None, out=None):
        """One decoder layer's linears for M tokens (input x, default self.x;
        fc2 output into `out`, default self.y['fc2']); returns this rank's fc2 shard."""
        x = self.x[:M] if x is None else x
        self._k1("q", x, M)
        cq, rq = self.codes["q"], self.rs["q"]
        # q / k / v share the input -> one launch over the three weight sets
        # (K5d for decode-shaped M, K5p stream-K over their pair tiles for prefill)
        self._k5_qkv(cq, rq, M)
        a = self._gather("q", M)  # attention-output stand-in, gathered for the out projection
        self._k1("out", a, M)
        self._k5("out", self.codes["out"], self.rs["out"], M)
        go = self._gather("out", M)
        self._k1("fc1", go, M)
        self._k5("fc1", self.codes["fc1"], self.rs["fc1"], M)
        g1 = self._gather("fc1", M)
        self._k1("fc2", g1, M)
        y2 = self.y["fc2"][:M] if out is None else out
        self._k5("fc2", self.codes["fc2"], self.rs["fc2"], M, out=y2)
        self._gather("fc2", M, src=y2)
        return y2


def verify_step(layer, M, n_rows=8):
    """Self-check of the timed work: sampled rows of this rank's fc1 and fc2
    outputs from the last step, against the reference's own dgq_forward
    (oracle/_ref, proj/src/kernel.cpp:144-153) on the same FP16 inputs
    (the gathered out / fc1 activations) and the rank's column shard.  The FP16
    output must equal fp16_round(reference FP32 output) bit for bit."""
    import numpy as np

    import oracle
    from paper_2310_04836_b200.parallel import gathered_to_full, shard_layer

    torch = __import__("torch")
    torch.cuda.synchronize()
    be = oracle.best()
    rows = np.unique(np.concatenate([[0, 255, 256, 511, M // 2, M - 1],
                                     np.random.default_rng(7).integers(0, M, n_rows - 6)]))
    res = {"rows": rows.tolist(), "oracle": be.kind}
    ok = True
    for name, src in (("fc1", "out"), ("fc2", "fc1")):
        g = layer.y[src][:M].unsqueeze(0) if layer.world == 1 else layer.g[src][:, :M]
        x = gathered_to_full(g)[torch.from_numpy(rows).to(g.device)].float().cpu().numpy()
        S = shard_layer(layer.host[name], layer.rank, layer.world) if layer.world > 1 else layer.host[name]
        out = be.dgq_forward(x, _oracle_layer(S), None, 0)[0] if be.kind == "reference" \
            else be.dgq_forward(x, _oracle_layer(S))[0]
        want = oracle.fp16_round_np(out).astype(np.float16).view(np.uint16)
        got = layer.y[name][torch.from_numpy(rows).to(g.device)].cpu().numpy().view(np.uint16)
        same = bool(np.array_equal(got, want))
        res[name] = {"bit_exact_fp16": same, "mismatches": int((got != want).sum()), "elements": int(got.size)}
        ok = ok and same
    res["ok"] = ok
    return res


def timed_steps(layer, M, steps, warmup, flush, sync_all, e2e=None):
    """Per-step CUDA-event times (s) with an L2 flush between steps; with e2e =
    (x_host, out_host) the step includes the H2D input copy and D2H output copy."""
    import torch

    def one():
        if e2e is not None:
            layer.x[:M].copy_(e2e[0], non_blocking=True)
        y = layer.step(M)
        if e2e is not None:
            e2e[1].copy_(y, non_blocking=True)

    for _ in range(warmup):
        one()
    sync_all()
    times = []
    for _ in range(steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        one()
        b.record()
        b.synchronize()
        times.append(a.elapsed_time(b) * 1e-3)
    sync_all()
    return times


def e2e_pipelined(layer, M, steps, warmup, x_hosts, out_hosts, sync_all):
    """End-to-end serving throughput through the public API: every step copies
    its f32 input from pinned host memory (x_hosts, alternating) and copies its
    fc2 output shard back to pinned host memory (out_hosts, alternating), on
    their own streams with double-buffered device tensors, so step i+1's input
    copy and step i-1's output copy run under step i's kernels (the serving
    pipeline).  Timed from the first input copy to the last output copy with CUDA
    events; returns seconds for `steps` steps (after `warmup` untimed ones)."""
    import torch

    dev = layer.x.device
    s_c = torch.cuda.current_stream(dev)
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    shard = layer.lin["fc2"].shard
    xd = [torch.empty(M, x_hosts[0].shape[1], dtype=torch.float32, device=dev) for _ in range(2)]
    od = [torch.empty(M, shard, dtype=torch.float16, device=dev) for _ in range(2)]
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_c = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]

    def run(n, t0=None, t1=None):
        for i in range(n):
            b = i % 2
            if i >= 2:
                s_in.wait_event(ev_c[b])  # step i-2 has consumed xd[b]
            if i == 0 and t0 is not None:
                t0.record(s_in)
            with torch.cuda.stream(s_in):
                xd[b].copy_(x_hosts[i % len(x_hosts)], non_blocking=True)
            ev_in[b].record(s_in)
            s_c.wait_event(ev_in[b])
            if i >= 2:
                s_c.wait_event(ev_out[b])  # step i-2's output left od[b]
            layer.step(M, x=xd[b], out=od[b])
            ev_c[b].record(s_c)
            s_out.wait_event(ev_c[b])
            with torch.cuda.stream(s_out):
                out_hosts[i % len(out_hosts)].copy_(od[b], non_blocking=True)
            ev_out[b].record(s_out)
        if t1 is not None:
            t1.record(s_out)

    run(warmup)
    sync_all()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    run(steps, t0, t1)
    t1.synchronize()
    sync_all()
    return t0.elapsed_time(t1) * 1e-3


def serving_call_detail(layer, M=SEQ):
    """The C-ABI serving call with host buffers (dgq_layer_forward_host, the
    reference-facing entry point a plugin binds): one OPT-30B linear per call,
    pinned host input and output, token chunks pipelined over copy streams.
    Wall-clock around the synchronous call (it includes the PCIe copies)."""
    import torch

    r = {}
    for name in ("q", "fc1", "fc2"):
        lin = layer.lin[name].layer
        xh = torch.from_numpy(_synth_x(M, lin.h)).pin_memory()
        yh = torch.empty(M, lin.o, dtype=torch.float16).pin_memory()
        X, Y = xh.numpy(), yh.numpy()
        import paper_2310_04836_b200 as dgq
        from paper_2310_04836_b200.api import _np_ptr, _stream

        def call():
            dgq._lib.check(dgq.lib().dgq_layer_forward_host(lin.handle, _np_ptr(X), M, None, 1, _np_ptr(Y),
                                                            _stream(lin.device)))
        call()
        best = 1e30
        for _ in range(5):
            t0 = time.perf_counter()
            call()
            best = min(best, time.perf_counter() - t0)
        ops = 2.0 * M * lin.h * lin.o
        r[name] = {"ms": round(best * 1e3, 3), "TOPS": round(ops / best / 1e12, 1),
                   "pcie_GBps": round((M * lin.h * 4 + M * lin.o * 2) / best / 1e9, 1)}
    return r


def _graph_of(fn):
    import torch

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()  # warm: allocates workspaces outside the capture
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
    torch.cuda.synchronize()
    return g


def decode_step_time(layer, M, flush, sync_all, world, reps=8):
    """Mean device time (s) of one decoder-layer step at M tokens."""
    import torch

    if world > 1:  # collectives stay eager under torchrun
        t = timed_steps(layer, M, reps, 2, flush, sync_all)
        return sum(t) / len(t)
    g = _graph_of(lambda: layer.step(M))
    times = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        times.append(a.elapsed_time(b) * 1e-3)
    return sum(times) / len(times)


def decode_k5_bandwidth(layer, M, flush, reps=8):
    """Algorithmic HBM GB/s of each K5 launch at M tokens (graph-replayed, L2 flushed)."""
    import torch

    out = {}
    for name, K, N in OPT30B:
        lin = layer.lin[name]
        key = "q" if name in ("q", "k", "v") else name
        codes, rs = layer.codes[key][:M], layer.rs[key][:M]
        g = _graph_of(lambda: lin.linear(codes, rs, out=layer.y[name][:M]))
        ts = []
        for _ in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e-3)
        t = sum(ts) / len(ts)
        ns = lin.shard
        byts = M * K + 4 * M + K * ns / 2 + (K / GROUP) * ns * 1.5 + 4 * ns + 2 * M * ns
        out[name] = byts / t / 1e9
    return out


def decode_k5_streaming(layer, M, device, world, group):
    """Steady-state algorithmic HBM GB/s of each distinct K5 shape at M tokens:
    one CUDA graph of back-to-back launches over R copies of the layer whose
    weights together exceed 2.2x L2 (every launch streams from HBM, as in a
    decoder stack), time / R.  Complements decode_k5_bandwidth (one launch
    after an L2 flush, which also carries the graph-launch latency)."""
    import torch

    from paper_2310_04836_b200.parallel import ColumnParallelLinear

    out = {}
    l2 = 126e6
    for name, K, N in (("q", 7168, 7168), ("fc1", 7168, 28672), ("fc2", 28672, 7168)):
        lin0 = layer.lin[name]
        wb = K * lin0.shard / 2 + (K / GROUP) * lin0.shard * 1.5
        copies = max(2, int(2.2 * l2 / wb) + 1)
        L = tiled_layer(K, N, seed=500)
        lins = [ColumnParallelLinear(L, int(os.environ.get("RANK", "0")), world, device, group)
                for _ in range(copies)]
        key = "q" if name in ("q", "k", "v") else name
        codes, rs = layer.codes[key][:M], layer.rs[key][:M]
        y = layer.y[name][:M]
        g = _graph_of(lambda: [ln.linear(codes, rs, out=y) for ln in lins])
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        t = a.elapsed_time(b) * 1e-3 / copies
        byts = M * K + 4 * M + wb + 4 * lin0.shard + 2 * M * lin0.shard
        out[name] = {"us": t * 1e6, "GBps": byts / t / 1e9, "copies": copies}
        del lins, g
        torch.cuda.empty_cache()
    return out


def measure_int8_peak(device):
    """Dense INT8 tensor throughput of this GPU: cuBLASLt (torch._int_mm), the
    best of 6 replays of a CUDA graph of 5 back-to-back calls on each of three
    shapes (8192^3, the OPT-30B fc1 shape, 4096x8192x8192) — a burst figure
    like MEASURED_PEAKS.json's bf16 one.  None if the library path is missing."""
    import torch

    try:
        top = 0.0
        for m, k, n in ((8192, 8192, 8192), (2048, 7168, 28672), (4096, 8192, 8192)):
            a = torch.randint(-127, 128, (m, k), dtype=torch.int8, device=device)
            b = torch.randint(-127, 128, (k, n), dtype=torch.int8, device=device)
            for _ in range(3):
                torch._int_mm(a, b)
            g = _graph_of(lambda: [torch._int_mm(a, b) for _ in range(5)])  # launch overhead amortised
            best = 1e30
            for _ in range(6):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                e1.synchronize()
                best = min(best, e0.elapsed_time(e1) * 1e-3 / 5)
            del a, b, g
            top = max(top, 2.0 * m * k * n / best / 1e12)
        return top
    except Exception:  # noqa: BLE001
        return None


def measure_tcgen05_i8_peak(sustained=False):
    """Dense INT8 tensor peak measured by this library's microbenchmark
    (dgq_measure_i8_peak: every SM pair issuing tcgen05.mma.cta_group::2.kind::i8
    256x256x32 back to back from shared memory): best of 10 launches (burst), or
    ~2500 launches back to back (~3 s) timed as one span (sustained: the clock
    the GPU holds under continuous tensor load)."""
    import ctypes

    import paper_2310_04836_b200 as dgq

    t, ms = ctypes.c_double(), ctypes.c_double()
    try:
        dgq._lib.check(dgq.lib().dgq_measure_i8_peak(-2500 if sustained else 10, ctypes.byref(t), ctypes.byref(ms)))
        return t.value
    except Exception:  # noqa: BLE001
        return None


def _stream_time(fns, reps=3):
    """Steady-state device time (s) per call of a list of launches replayed from
    one CUDA graph (callers rotate over weight copies larger than L2, so every
    launch streams its weights from HBM)."""
    import torch

    g = _graph_of(lambda: [f() for f in fns])
    g.replay()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b) * 1e-3 / len(fns))
    del g
    return best


def k5_bytes(M, K, N, g=GROUP):
    """Algorithmic HBM bytes of one K5 launch, FP16 output."""
    return M * K + 4 * M + K * N / 2 + (K / g) * N * 1.5 + 4 * N + 2 * M * N


def linear_point(K, N, Ms, device, hbm_peak, i8_peak, g=GROUP, shard=None, seed=900):
    """Per-M steady-state time of one DGQ linear (K1 excluded): weights rotated
    through copies totalling > 2.2x L2, launches replayed from a CUDA graph.
    Returns {M: {us, TOPS, GBps, bound, frac}} with the bound (HBM or INT8
    tensor) the larger of the two roofline times."""
    import torch

    import paper_2310_04836_b200 as dgq

    L = tiled_layer(K, N, seed=seed, group=g)
    c0, c1 = shard if shard else (0, N)
    n = c1 - c0
    wb = K * n / 2 + (K / g) * n * 1.5
    copies = max(2, int(2.2 * 126e6 / wb) + 1)
    layers = [dgq.CudaLayer(L, device=device, col_begin=c0, col_end=c1, validate=(i == 0)) for i in range(copies)]
    out = {}
    for M in Ms:
        x = torch.from_numpy(_synth_x(M, K)).to(device)
        codes, rs = layers[0].quantize_act(x)
        y = torch.empty(M, n, dtype=torch.float16, device=device)
        t = _stream_time([lambda Lc=Lc: Lc.linear(codes, rs, out=y) for Lc in layers])
        ops, byts = 2.0 * M * K * n, k5_bytes(M, K, n, g)
        t_hbm, t_i8 = byts / (hbm_peak * 1e9), ops / (i8_peak * 1e12)
        bound = "hbm" if t_hbm >= t_i8 else "tensor"
        out[M] = {"us": round(t * 1e6, 2), "TOPS": round(ops / t / 1e12, 1), "GBps": round(byts / t / 1e9),
                  "bound": bound, "frac": round(max(t_hbm, t_i8) / t, 3), "plan": layers[0].plan(M)}
        del x, codes, rs, y
    del layers
    torch.cuda.empty_cache()
    return out


def _synth_x(M, K):
    from paper_2310_04836_b200 import synth

    return synth.gen_synthetic(M, K, 101 + M, 3, 50.0, 7)


def k1_point(M, K, f16, device, hbm_peak):
    """K1 standalone: steady-state GB/s over input copies > 2.2x L2."""
    import torch

    from paper_2310_04836_b200 import CudaLayer, synth

    L = tiled_layer(K, 512, seed=77)
    L.k = synth.smooth_k(K)
    CL = CudaLayer(L, device=device)
    x0 = torch.from_numpy(_synth_x(M, K)).to(device)
    if f16:
        x0 = x0.half()
    nb = x0.numel() * x0.element_size()
    xs = [x0.clone() for _ in range(max(2, int(2.2 * 126e6 / nb) + 1))]
    codes, rs = CL.quantize_act(x0)
    t = _stream_time([lambda x=x: CL.quantize_act(x, codes, rs) for x in xs])
    byts = M * K * (2 if f16 else 4) + 4 * K + M * K + 4 * M
    del xs
    torch.cuda.empty_cache()
    return {"us": round(t * 1e6, 2), "GBps": round(byts / t / 1e9), "hbm_frac": round(byts / t / 1e9 / hbm_peak, 3)}


def config_sweeps(device, hbm_peak, i8_peak):
    """The BASELINE.json configs beyond the headline step."""
    r = {}
    # C1 + C5: M sweep on K = N = 4096, g in {64, 128}
    Ms = [1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 8192]
    r["C5_4096x4096_g128"] = linear_point(4096, 4096, Ms, device, hbm_peak, i8_peak, g=128)
    r["C5_4096x4096_g64"] = linear_point(4096, 4096, [1, 16, 256, 2048], device, hbm_peak, i8_peak, g=64)
    # C2: LLaMA-7B layer GEMMs, prefill M = 2048 and decode M = 1
    for name, K, N in (("qkv_o", 4096, 4096), ("up_gate", 4096, 11008), ("down", 11008, 4096)):
        r[f"C2_llama7b_{name}"] = linear_point(K, N, [2048, 1], device, hbm_peak, i8_peak)
    # C4: LLaMA-65B FFN on one 8-way column shard, decode batch 1-64
    for name, K, N in (("up", 8192, 22016), ("down", 22016, 8192)):
        w = N // 8
        r[f"C4_llama65b_{name}_shard8"] = linear_point(K, N, [1, 2, 4, 8, 16, 32, 64], device, hbm_peak, i8_peak,
                                                       shard=(3 * w, 4 * w))
    # C5: K1 standalone
    r["C5_k1"] = {f"M{M}_K{K}_{'f16' if f else 'f32'}": k1_point(M, K, f, device, hbm_peak)
                  for M, K, f in ((2048, 7168, False), (2048, 7168, True), (2048, 28672, True), (16, 4096, False),
                                  (8192, 4096, False))}
    return r


def _graph_time(fn, flush, reps=6):
    """Mean device time (s) of fn replayed from a CUDA graph, L2 flushed before each replay."""
    import torch

    g = _graph_of(fn)
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    return sum(ts) / len(ts)


def _marlin_a16w4(K, N, device):
    """A fused weight-only INT4 GEMM (A16W4, group 128, FP16 activations): vLLM's
    Marlin kernel (library code, the standard W4A16 kernel) on the same shape.
    Returns a callable x16 -> y16, or raises when vLLM / its kernels are absent."""
    import torch
    import vllm._custom_ops as ops
    from vllm.model_executor.layers.quantization.utils.marlin_utils import marlin_make_workspace_new
    from vllm.model_executor.layers.quantization.utils.marlin_utils_test import marlin_quantize
    from vllm.scalar_type import scalar_types

    w = torch.randn(K, N, dtype=torch.float16, device=device) * 0.02
    _, q_w, s, g_idx, sort_idx, _ = marlin_quantize(w, scalar_types.uint4b8, GROUP, False)
    ws = marlin_make_workspace_new(device)
    del w

    def run(x16):
        return ops.marlin_gemm(x16, None, q_w, None, s, None, None, None, g_idx, sort_idx, ws, scalar_types.uint4b8,
                               size_m=x16.shape[0], size_n=N, size_k=K, is_k_full=True)
    return run


def comparators(layer, flush):
    """the paper's comparisons on B200 for OPT-30B fc1
    (7168 -> 28672) — DGQ A8W4 (this repo) against library baselines on the same
    GPU: A8W8 (cuBLASLt int8, torch._int_mm on the dequantised int8 weights),
    A16W16 (cuBLAS fp16) and A16W4 weight-only (dequantise the INT4 layer to
    fp16 each call, then cuBLAS fp16).  TOPS = 2*M*N*K / device time."""
    import torch

    lin = layer.lin["fc1"]
    K, N = lin.h, lin.shard
    out = {}
    try:
        marlin = _marlin_a16w4(K, N, layer.x.device)
    except Exception as e:  # noqa: BLE001
        marlin, marlin_err = None, f"unavailable: {type(e).__name__}: {str(e)[:120]}"
    w8 = lin.layer.dequant_s8()[:K, :N].contiguous()            # [K, N] int8
    s1 = torch.full((N,), 1.0 / (32.0 * K ** 0.5), device=w8.device)  # per-channel scale (values do not affect timing)
    w16 = (w8.to(torch.float16) * s1.to(torch.float16))         # A16W16 weights
    for M in (2048, 32):
        ops = 2.0 * M * N * K
        codes, rs = layer.codes["fc1"][:M], layer.rs["fc1"][:M]
        y = layer.y["fc1"][:M]
        r = {"dgq_a8w4": ops / _graph_time(lambda: lin.linear(codes, rs, out=y), flush) / 1e12}
        xq = codes[:, :K].contiguous()
        try:
            r["a8w8_cublaslt"] = ops / _graph_time(lambda: torch._int_mm(xq, w8), flush) / 1e12
        except Exception as e:  # noqa: BLE001
            r["a8w8_cublaslt"] = f"unavailable: {type(e).__name__}"
        x16 = torch.randn(M, K, device=w8.device, dtype=torch.float16)
        r["a16w16_cublas"] = ops / _graph_time(lambda: x16 @ w16, flush) / 1e12

        def a16w4():
            wq = lin.layer.dequant_s8()
            return x16 @ (wq[:K, :N].to(torch.float16) * s1.to(torch.float16))
        # a labelled LOWER bound only (dequantise the whole layer every call); the
        # fair weight-only comparator is the fused Marlin kernel below
        r["a16w4_dequant_then_cublas_lower_bound"] = ops / _graph_time(a16w4, flush) / 1e12
        if marlin is not None:
            try:
                r["a16w4_marlin_fused"] = ops / _graph_time(lambda: marlin(x16), flush) / 1e12
                r["dgq_speedup_vs_a16w4"] = r["dgq_a8w4"] / r["a16w4_marlin_fused"]
            except Exception as e:  # noqa: BLE001
                r["a16w4_marlin_fused"] = f"unavailable: {type(e).__name__}: {str(e)[:120]}"
        else:
            r["a16w4_marlin_fused"] = marlin_err
        if isinstance(r["a8w8_cublaslt"], float):
            r["dgq_speedup_vs_a8w8"] = r["dgq_a8w4"] / r["a8w8_cublaslt"]
        out[f"fc1_M{M}_TOPS"] = r
    out["weight_bytes_fc1"] = {"a8w4_dgq": K * N / 2 + (K / GROUP) * N * 1.5, "a8w8": K * N, "a16w16": 2 * K * N}
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=device)

    def sync_all():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    import paper_2310_04836_b200 as dgq

    dgq.lib()
    hbm_peak, bf16_peak, peak_src = load_peaks()
    i8_proxy = 2.0 * bf16_peak  # dense INT8 = 2x dense BF16 (FP8-class rate); spec 4500
    i8_cublas = measure_int8_peak(device)  # cuBLASLt int8 burst on this GPU
    i8_tc = measure_tcgen05_i8_peak()  # tcgen05 kind::i8 microbenchmark, burst (best of 10)
    # the K5 launches are timed inside a long step: the roofline denominator is
    # the SUSTAINED rate (~3 s back to back: the clock the GPU holds under
    # continuous tensor load), the burst figure is reported beside it
    i8_tc_sus = measure_tcgen05_i8_peak(sustained=True)
    i8_peak = i8_tc_sus or i8_tc or max(i8_proxy, i8_cublas or 0.0)
    layer = OptLayer(rank, world, device, group, SEQ)
    torch.manual_seed(1234 + 0)
    # the reference's synthetic activations: N(0, 1) with three
    # outlier channels x50 (column seed 7, the channels smooth_k scales down)
    from paper_2310_04836_b200 import synth
    x_host = torch.from_numpy(synth.gen_synthetic(SEQ, 7168, 101, 3, 50.0, 7)).pin_memory()
    layer.x.copy_(x_host)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device)
    sync_all()

    # ---- headline: device-resident step at seq 2048 ------------------------------------------
    clocks = ClockSampler(torch.cuda.current_device() if "CUDA_VISIBLE_DEVICES" not in os.environ else local)
    layer.record = False
    for _ in range(args.warmup):
        layer.step(SEQ)
    sync_all()
    clocks.start()
    times = timed_steps(layer, SEQ, args.steps, 0, flush, sync_all)
    clk = clocks.stop()
    # per-launch CUDA events (roofline, per-kernel detail) in a second pass of
    # the same K steps: an event recorded between two launches chained by
    # programmatic dependent launch serialises them (the next kernel can no
    # longer start while the previous one drains), so the headline pass above
    # carries only the step's own events
    layer.record = True
    timed_steps(layer, SEQ, args.steps, 0, flush, sync_all)
    layer.record = False
    total = max_over_ranks(sum(times))
    ops_step = layer_ops(SEQ)
    value = ops_step * args.steps / total / 1e12
    ms_per_step = total / args.steps * 1e3

    # roofline of the dominant kernel (K5), measured over the timed region
    k5_t = sum(a.elapsed_time(b) * 1e-3 for a, b, _, _ in layer.k_events)
    k5_ops = sum(o for _, _, o, _ in layer.k_events)
    k5_tops = k5_ops / k5_t / 1e12
    by_name = {}
    for a, b, o, n in layer.k_events:
        t, oo = by_name.get(n, (0.0, 0.0))
        by_name[n] = (t + a.elapsed_time(b) * 1e-3, oo + o)
    k1_by = {}
    for a, b, bb, n in layer.q_events:
        t, x = k1_by.get(n, (0.0, 0.0))
        k1_by[n] = (t + a.elapsed_time(b) * 1e-3, x + bb)
    k1_t = sum(a.elapsed_time(b) * 1e-3 for a, b, _, _ in layer.q_events)
    k1_b = sum(bb for _, _, bb, _ in layer.q_events)
    n_launches = len(layer.k_events) + len(layer.q_events)
    # DRAM traffic of the K5 launches from the committed ncu captures (one
    # `ncu --set full` launch per shape, tools/profile_r02.sh): average bytes per
    # launch over the step's four K5 launches (the out projection has q's shape)
    traffic, traffic_by = None, None
    prof = os.path.join(ROOT, "profiles", "ncu_summary_r02i.json")
    if os.path.exists(prof) and world == 1:
        try:
            pr = json.load(open(prof))

            def _db(k):
                return (float(pr[k]["dram__bytes_read.sum"]) + float(pr[k]["dram__bytes_write.sum"])) * 1e6
            traffic_by = {"qkv": _db("k5p_qkv"), "out": _db("k5p_q"), "fc1": _db("k5p_fc1"), "fc2": _db("k5p_fc2")}
            traffic = sum(traffic_by.values()) / 4
        except Exception:
            traffic, traffic_by = None, None

    # ---- self-check of the timed outputs (after the timed region) ---------------------------
    try:
        verified = verify_step(layer, SEQ)
    except Exception as e:  # noqa: BLE001  (oracle not built on this box)
        verified = {"ok": None, "error": f"{type(e).__name__}: {e}"}

    # ---- e2e through the public API with host buffers ---------------------------------------
    x_hosts = [x_host, x_host.clone().pin_memory()]
    out_hosts = [torch.empty(SEQ, layer.lin["fc2"].shard, dtype=torch.float16).pin_memory() for _ in range(2)]
    e2e_total = max_over_ranks(e2e_pipelined(layer, SEQ, args.steps, max(1, args.warmup), x_hosts, out_hosts,
                                             sync_all))
    e2e_val = ops_step * args.steps / e2e_total / 1e12
    # the same step with the copies serialised with the kernels (no pipelining), for reference
    e2e_serial = timed_steps(layer, SEQ, max(3, args.steps // 2), 1, flush, sync_all,
                             e2e=(x_host, out_hosts[0]))
    e2e_serial_val = ops_step * len(e2e_serial) / max_over_ranks(sum(e2e_serial)) / 1e12

    # ---- detail: layer ms at seq 512 / 1024, decode (M = 16) weight bandwidth ----------------
    detail = {}
    if not args.no_detail:
        try:
            for M in (512, 1024):
                t = timed_steps(layer, M, 3, 1, flush, sync_all)
                tm = max_over_ranks(sum(t)) / 3
                detail[f"layer_ms_seq{M}"] = tm * 1e3
                detail[f"tops_seq{M}"] = layer_ops(M) / tm / 1e12
            detail["layer_ms_seq2048"] = ms_per_step
            for M in (1, 16):
                # decode steps are launch-bound from Python: replay the step from a CUDA graph
                # (single rank) so the number is the GPU's; L2 flushed before every replay
                tm = decode_step_time(layer, M, flush, sync_all, world)
                tm = max_over_ranks(tm)
                wb = layer_weight_bytes(world)
                detail[f"decode_m{M}_layer_us"] = tm * 1e6
                detail[f"decode_m{M}_weight_GBps_per_gpu"] = wb / tm / 1e9
                detail[f"decode_m{M}_hbm_frac"] = wb / tm / 1e9 / hbm_peak
                if world == 1:
                    kb = decode_k5_bandwidth(layer, M, flush)
                    detail[f"decode_m{M}_k5_GBps"] = kb
                    detail[f"decode_m{M}_k5_hbm_frac"] = {n: v / hbm_peak for n, v in kb.items()}
                    try:
                        st = decode_k5_streaming(layer, M, device, world, group)
                        detail[f"decode_m{M}_k5_streaming"] = {n: dict(v, hbm_frac=v["GBps"] / hbm_peak)
                                                              for n, v in st.items()}
                    except Exception as e:  # noqa: BLE001
                        detail[f"decode_m{M}_k5_streaming"] = {"error": f"{type(e).__name__}: {e}"}
            detail["k5_tops_by_linear"] = {n: o / t / 1e12 for n, (t, o) in by_name.items()}
            if traffic_by:
                alg = {n: k5_bytes(SEQ, K, N // world) for n, K, N in (("out", 7168, 7168), ("fc1", 7168, 28672),
                                                                         ("fc2", 28672, 7168))}
                # the fused q/k/v launch reads the shared codes and row scales once
                alg["qkv"] = 3 * alg["out"] - 2 * (SEQ * 7168 + 4 * SEQ)
                detail["k5_dram_bytes_by_linear"] = {n: {"ncu_dram_bytes": traffic_by[n], "algorithmic_bytes": alg[n],
                                                         "ratio": round(traffic_by[n] / alg[n], 2)} for n in alg}
            detail["k1_GBps"] = k1_b / k1_t / 1e9
            detail["k1_GBps_by_input"] = {n: x / t / 1e9 for n, (t, x) in k1_by.items()}
            plans = {n: layer.lin[n].layer.plan(SEQ) for n in ("q", "fc1", "fc2")}
            detail["plans_seq2048"] = plans
            if world == 1:
                try:
                    detail["comparators"] = comparators(layer, flush)
                except Exception as e:  # noqa: BLE001  (a library baseline must not sink the bench line)
                    detail["comparators"] = {"error": f"{type(e).__name__}: {e}"}
                try:
                    detail["serving_call_host_buffers"] = serving_call_detail(layer)
                except Exception as e:  # noqa: BLE001
                    detail["serving_call_host_buffers"] = {"error": f"{type(e).__name__}: {e}"}
                try:
                    detail["configs"] = config_sweeps(device, hbm_peak, i8_peak)
                except Exception as e:  # noqa: BLE001
                    detail["configs"] = {"error": f"{type(e).__name__}: {e}"}
            detail["peaks"] = {"hbm_GBps": hbm_peak, "i8_tcgen05_TOPS": i8_tc, "i8_tcgen05_sustained_TOPS": i8_tc_sus,
                               "i8_cublaslt_TOPS": i8_cublas,
                               "i8_2x_bf16_TOPS": i8_proxy}
        except Exception as e:  # noqa: BLE001  (a detail probe must never sink the headline line)
            detail["error"] = f"{type(e).__name__}: {e}"

    cpu = None
    if rank == 0 and not args.no_cpu:
        try:
            cpu = cpu_baseline_sample()
        except Exception as e:  # oracle not built on this box
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "unavailable", "sample": str(e)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "int8 (i8 x i8 -> i32 tcgen05 kind::i8; fp32 scales; fp16 out)",
            "data": "synthetic (random valid DGQ layers with the reference's compute_smooth k; the reference's gen_synthetic activations, 3 outlier channels x50)",
            "config": {
                "workload": "OPT-30B decoder-layer linears (q,k,v,out 7168x7168; fc1 7168x28672; fc2 28672x7168) "
                            "+ 4 activation quantisations, seq 2048, g=128, FP16 out",
                "seq_len": SEQ, "group": GROUP, "parallelism": f"column-parallel N-shard x{world} (NCCL all-gather)",
                "l2": "flushed between timed steps (256 MiB write); per-GPU weights "
                      f"{layer_weight_bytes(world) / 1e6:.0f} MB",
            },
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": SEQ * 7168 * 4,
                    "d2h_bytes_per_step": SEQ * layer.lin["fc2"].shard * 2, "per": "rank",
                    "pipeline": "input copy of step i+1 and output copy of step i-1 on their own streams under "
                                "step i's kernels (double-buffered device tensors, pinned host buffers)",
                    "serialised_value": e2e_serial_val},
            "gpu_launches": n_launches,
            "roofline": {"bound": "tensor", "kernel": "K5 fused DGQ linear (all four launches per step: qkv, out, fc1, fc2)",
                         "achieved": k5_tops, "peak": i8_peak, "unit": "TFLOP/s", "frac": k5_tops / i8_peak,
                         "peak_note": (f"measured here: tcgen05.mma.cta_group::2.kind::i8 microbenchmark "
                                       f"(dgq_measure_i8_peak) sustained over ~3 s back to back = "
                                       f"{(i8_tc_sus or 0.0):.0f} TOPS (the K5 launches run inside a long step); "
                                       f"burst (best of 10) {(i8_tc or 0.0):.0f} TOPS (frac "
                                       f"{k5_tops / (i8_tc or 1e30):.3f}); "
                                       f"also cuBLASLt int8 burst {(i8_cublas or 0.0):.0f} TOPS (frac "
                                       f"{k5_tops / (i8_cublas or 1e30):.3f}), 2 x bf16 {i8_proxy:.0f} "
                                       f"({peak_src}), NVIDIA spec dense INT8 4500 (frac {k5_tops / 4500:.3f})"),
                         "achieved_how": "2*M*N*K of each K5 launch / its CUDA-event time, averaged over the "
                                         "launches of a second pass of the same K steps (per-launch events would "
                                         "serialise the PDL-chained launches of the headline pass)",
                         "traffic": traffic},
            "cpu_baseline": cpu,
            "verified": verified.get("ok"),
            "verification": verified,
            "clocks": clk,
            "detail": detail,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-detail", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
