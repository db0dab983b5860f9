"""Whole-model layer-wise sweep across the GPUs of one box (BASELINE.json
configs[3], C4): 32 Llama-2-7B-shaped decoder blocks x 7 linears, W4 g128,
act-order, 262144 calibration tokens per tap, total wall-clock reported.

Reference: run_layerwise_sweep (pipeline.cpp:185-280) visits the model's
layers one by one -- collect the layer's inputs, accumulate_stats,
quantize_layer -- and q/k/v read the same attention input and gate/up the
same MLP input (model.cpp:301-307).  Here the unit of work is one DISTINCT
calibration input ("tap"): 4 per block (attn_in -> q, k, v; o_in -> o;
mlp_in -> gate, up; down_in -> down), 128 in the model.  A unit is one
Hessian + one order/factorisation (they depend on H only, layerwise.cpp:29-51)
and one grid + sweep + pack per linear that reads the tap
(ocwg_quantize_layers_x_dev).

With synthetic calibration data the units are independent (no model forward
between layers), so they are spread over the ranks by LPT (longest
processing time first) on a cost model of the hot path's phases (SURVEY
Appendix B work terms at measured rates): a down_proj unit (N = 11008) weighs
about 5x an attention unit.  Each rank generates its units' X and W on the
device (synth.cu, the seeds of SURVEY §8(d)), quantizes them, and keeps the
packed OCW1 payloads; rank 0 can gather every payload over NCCL (P2P sends).

Orientation is the reference's: W is N (in) x M (out).
"""
from __future__ import annotations

import heapq
from dataclasses import dataclass

HIDDEN, FFN, BLOCKS, TOKENS = 4096, 11008, 32, 262144
CFG_INDEX = 3  # BASELINE.json configs[3]
TAPS = ("attn_in", "o_in", "mlp_in", "down_in")


@dataclass(frozen=True)
class Unit:
    """One distinct calibration input and the linears that read it."""
    block: int
    tap: str
    n: int                   # input channels (rows of every W)
    linears: tuple           # ((name, M), ...)
    silu: bool               # down_proj input: SiLU(a) * b

    @property
    def index(self) -> int:  # tap number in model order
        return 4 * self.block + TAPS.index(self.tap)

    def layer_index(self, k: int) -> int:  # linear number in model order (7 per block)
        base = {"attn_in": 0, "o_in": 3, "mlp_in": 4, "down_in": 6}[self.tap]
        return 7 * self.block + base + k


def model_units(blocks: int = BLOCKS, hidden: int = HIDDEN, ffn: int = FFN) -> list[Unit]:
    """The 4 taps of each block in model order (model.cpp:301-307)."""
    out = []
    for b in range(blocks):
        out.append(Unit(b, "attn_in", hidden, (("q_proj", hidden), ("k_proj", hidden),
                                               ("v_proj", hidden)), False))
        out.append(Unit(b, "o_in", hidden, (("o_proj", hidden),), False))
        out.append(Unit(b, "mlp_in", hidden, (("gate_proj", ffn), ("up_proj", ffn)), False))
        out.append(Unit(b, "down_in", ffn, (("down_proj", hidden),), True))
    return out


def unit_cost(u: Unit, tokens: int = TOKENS) -> float:
    """Estimated seconds on one B200: Hessian F_H = T N (N+1) at ~1.25 PF/s,
    factorisation ~1.1 ms x (N/4096)^2 (a latency chain over N/64 tile
    columns), per linear the in-block chain (~35 us per 128 rows per 4736
    columns) plus the 3xTF32 trailing GEMMs (2 N^2 M at ~300 TF/s)."""
    n = u.n
    t = tokens * n * (n + 1) / 1.25e15 + 1.1e-3 * (n / 4096) ** 2
    for _, m in u.linears:
        t += (n / 128) * 35e-6 * -(-m // 4736) + 2.0 * n * n * m / 3e14
    return t


def lpt(units: list[Unit], world: int, tokens: int = TOKENS) -> list[list[Unit]]:
    """Longest processing time first: units by descending cost (model order on
    ties) onto the least-loaded rank (lowest rank on ties).  Each rank's list
    is returned in model order."""
    order = sorted(range(len(units)), key=lambda i: (-unit_cost(units[i], tokens), i))
    heap = [(0.0, r) for r in range(world)]
    plan: list[list[int]] = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        plan[r].append(i)
        heapq.heappush(heap, (load + unit_cost(units[i], tokens), r))
    return [[units[i] for i in sorted(p)] for p in plan]


def seeds(u: Unit) -> dict:
    """W 0x5EED0000 + 16 cfg + layer, X 0x5EED1000 + 16 cfg + tap,
    outlier pick 0x5EED2000 + cfg (the residual stream's outlier channels are
    shared by the hidden-width taps)."""
    return {"x": 0x5EED1000 + 16 * CFG_INDEX + u.index,
            "w": [0x5EED0000 + 16 * CFG_INDEX + u.layer_index(k) for k in range(len(u.linears))],
            "pick": 0x5EED2000 + CFG_INDEX}


def outlier_scale(n: int, frac: float, seed: int, osc: float):
    """Per-channel scale: round(frac n) channels (seeded Fisher-Yates) x osc."""
    import numpy as np
    k = int(round(frac * n))
    rng = np.random.default_rng(seed)
    perm = np.arange(n)
    for i in range(n - 1, n - 1 - k, -1):
        j = int(rng.integers(0, i + 1))
        perm[i], perm[j] = perm[j], perm[i]
    s = np.ones(n, np.float32)
    s[perm[n - k:]] = osc
    return s


def run_rank(units: list[Unit], device: int, tokens: int = TOKENS, bits: int = 4, group: int = 128,
             keep_payload: bool = True, timing: bool = True, overlap: bool | None = None):
    """Quantize this rank's units on `device`.  Returns (payloads {layer name:
    uint8 device tensor}, stats) -- stats has the device time of the whole
    loop (CUDA events) and the unit count / weights.

    With overlap (OCWG_MODEL_OVERLAP=1) the calibration X of unit k+1 is
    generated on a second, lower-priority stream into the other half of a
    double buffer while unit k is quantized.  Measured on one B200 it gains
    nothing (3.19 s vs 3.21 s for the 32-block model): the generator only
    finds room beside the Hessian, which it slows down, as the factorisation
    fills every SM's register file.  So the default is sequential, which
    also separates the generation (a stand-in for the model forward that
    collects layer inputs) from the quantization in the stats."""
    import torch

    from . import GptqOptions, Granularity, QuantConfig, Scheme, dev

    import os
    if overlap is None:
        overlap = os.environ.get("OCWG_MODEL_OVERLAP", "0") == "1"
    cfg = QuantConfig(bits, Scheme.asymmetric, Granularity.per_group, group)
    opts = GptqOptions(actorder=True, percdamp=0.01, block_cols=128)
    dv = torch.device("cuda", device)
    payloads = {}
    stats = {"units": len(units), "weights": 0, "ms": 0.0, "overlap": overlap}
    if not units:
        return payloads, stats
    nmax = max(u.n for u in units)
    nbuf = 2 if overlap else 1
    xbuf = [torch.empty(tokens * nmax, dtype=torch.bfloat16, device=dv) for _ in range(nbuf)]
    scales = {}
    for u in units:
        if not u.silu and u.n not in scales:
            scales[u.n] = torch.from_numpy(outlier_scale(u.n, 0.01, seeds(u)["pick"], 20.0)).to(dv)
    # the quantization on a high-priority stream, the generator at default priority:
    # pending factorisation / sweep CTAs are dispatched before further generator CTAs
    main = torch.cuda.Stream(dv, priority=-5) if overlap else torch.cuda.current_stream(dv)
    gen = torch.cuda.Stream(dv) if overlap else main
    torch.cuda.synchronize(dv)
    ready = [torch.cuda.Event() for _ in range(nbuf)]
    free = [torch.cuda.Event() for _ in range(nbuf)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # per-unit phase events (meaningful without overlap): generation | quantization
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in units]

    def xview(k):
        u = units[k]
        return xbuf[k % nbuf][:tokens * u.n].view(tokens, u.n)

    def gen_x(k):
        u = units[k]
        with torch.cuda.stream(gen):
            if k >= nbuf:
                gen.wait_event(free[k % nbuf])
            if u.silu:
                dev.synth(1, seeds(u)["x"], xview(k))
            else:
                dev.synth(0, seeds(u)["x"], xview(k), col_scale=scales[u.n])
            ready[k % nbuf].record(gen)

    dev.set_async(True, device)  # device calls only enqueue; errors surface at synchronize
    ctx_main = torch.cuda.stream(main)
    ctx_main.__enter__()
    t0.record(main)
    if overlap:
        gen.wait_event(t0)
    for k in range(min(nbuf, len(units))):
        gen_x(k)
    for k, u in enumerate(units):
        sd = seeds(u)
        main.wait_event(ready[k % nbuf])
        ev[k][0].record(main)
        ws, outs = [], []
        for (name, m), wseed in zip(u.linears, sd["w"]):
            w = torch.empty((u.n, m), dtype=torch.float32, device=dv)
            dev.synth(2, wseed, w, stddev=0.02)
            ws.append(w)
            outs.append(dev.LayerBuffers(u.n, m, cfg, device, w_hat=False, payload=keep_payload, h=False))
            stats["weights"] += u.n * m
        dev.quantize_layers(ws, xview(k), cfg, opts, outs)
        ev[k][1].record(main)
        free[k % nbuf].record(main)
        if k + nbuf < len(units):
            gen_x(k + nbuf)
        for (name, m), o in zip(u.linears, outs):
            if keep_payload:
                payloads[f"model.layers.{u.block}.{name}"] = o.payload
        del ws, outs
    t1.record(main)
    ctx_main.__exit__(None, None, None)
    torch.cuda.synchronize(dv)
    try:
        dev.synchronize(device)
    finally:
        dev.set_async(False, device)
    if timing:
        stats["ms"] = t0.elapsed_time(t1)
        # W synthesis + Hessian + factorisation + sweeps + pack per unit (the
        # X generation, which stands in for the model forward, is the rest)
        stats["quant_ms"] = sum(a.elapsed_time(b) for a, b in ev)
        stats["gen_ms"] = stats["ms"] - stats["quant_ms"] if not overlap else None
    return payloads, stats


def layer_names(u: Unit) -> list[str]:
    return [f"model.layers.{u.block}.{name}" for name, _ in u.linears]


def gather_payloads(plan: list[list[Unit]], payloads: dict, payload_bytes, group=None) -> dict | None:
    """Every rank's packed payloads to rank 0 (point-to-point: NCCL over
    NVLink on the GPUs, gloo on CPU).  The plan is deterministic, so rank 0
    knows which layers each rank holds and their sizes (payload_bytes(n, m)):
    no header exchange.  Returns {layer name: uint8 tensor} on rank 0, None
    elsewhere."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if rank != 0:
        reqs = [dist.isend(payloads[name].contiguous(), dst=0, group=group)
                for u in plan[rank] for name in layer_names(u)]
        for r in reqs:
            r.wait()
        return None
    out = dict(payloads)
    dv = next(iter(payloads.values())).device if payloads else torch.device("cpu")
    reqs = []
    for r in range(1, world):
        for u in plan[r]:
            for (name, m), key in zip(u.linears, layer_names(u)):
                buf = torch.empty(payload_bytes(u.n, m), dtype=torch.uint8, device=dv)
                reqs.append(dist.irecv(buf, src=r, group=group))
                out[key] = buf
    for q in reqs:
        q.wait()
    return out
