#!/usr/bin/env python
"""Benchmark: GPTQ layer quantize of BASELINE.json configs[1] (C2) on B200.

Workload (reference orientation): W 4096 (in) x 4096 (out),
bf16-valued ~N(0, 0.02^2); calibration X = 128 x 2048 = 262144 tokens x 4096
bf16 ~N(0,1) with 1% of input channels (41, seeded Fisher-Yates) scaled x20;
4-bit asymmetric, group 128, act-order, percdamp 0.01, block 128.

One step = the whole hot path on one layer: H = X^T X (tcgen05 SYRK) ->
dampen/permute/factorise -> GPTQ sweep (codes, fp16-rounded scales, zeros,
W_hat) -> OCW1 payload pack.  Inputs are device resident and larger than L2
(X is 2 GiB), so no L2 flush is needed between steps.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

N > 1 (torchrun), --mode layers (default): every rank quantizes its own layer (weak scaling, no data-
path collective -- layers are independent; BASELINE configs 3-5's token-
sharded Hessian path is exercised by tests and `--mode sharded`).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N_IN, M_OUT, TOKENS, BITS, GROUP = 4096, 4096, 128 * 2048, 4, 128
SEED_W, SEED_X, SEED_PICK = 0x5EED0000 + 16 * 2, 0x5EED1000 + 16 * 2, 0x5EED2000 + 2
METRIC = "GPTQ layer quantize throughput (weights/s), 4096x4096 W4 g128, 262144 calib tokens"
F_H = TOKENS * N_IN * (N_IN + 1)                     # symmetric Hessian flops
F_FACT = 2 * N_IN ** 3 / 3
F_SWEEP = N_IN * (N_IN - 1) * M_OUT


def peaks():
    """(bf16 TF/s burst, bf16 TF/s sustained, HBM GB/s, source).  The timed loop
    lasts well under the seconds-long sustained measurement, so the Hessian's
    roofline uses the burst figure (the sustained fraction is reported beside)."""
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        burst = d.get("bf16_tflops", 1597.8)
        return burst, d.get("bf16_tflops_sustained", burst), d.get("hbm_gbs", 6548.8), "measured"
    return 1590.0, 1590.0, 6650.0, "fallback"


# DRAM bytes (read + write) of one hessian_tc2_kernel launch at C2, from the
# ncu --set full capture of gram_tc_kernel in profiles/r02_gram_ncu_full.txt
HESSIAN_TRAFFIC_BYTES = 4665406000 + 622313728  # ncu dram read + write, one C2 launch (profiles/r02_gram_ncu_full.txt)


def outlier_channels(n: int, frac: float, seed: int) -> np.ndarray:
    """Seeded Fisher-Yates pick of round(frac*n) channels."""
    k = int(round(frac * n))
    rng = np.random.default_rng(seed)
    perm = np.arange(n)
    for i in range(n - 1, n - 1 - k, -1):
        j = int(rng.integers(0, i + 1))
        perm[i], perm[j] = perm[j], perm[i]
    return np.sort(perm[n - k:])


def make_inputs(device, torch):
    g = torch.Generator(device=device)
    g.manual_seed(SEED_W)
    w = (torch.randn(N_IN, M_OUT, generator=g, device=device) * 0.02).to(torch.bfloat16).float()
    g.manual_seed(SEED_X)
    x = torch.empty(TOKENS, N_IN, dtype=torch.bfloat16, device=device)
    scale = torch.ones(N_IN, device=device)
    scale[torch.from_numpy(outlier_channels(N_IN, 0.01, SEED_PICK)).to(device)] = 20.0
    chunk = 16384
    for t0 in range(0, TOKENS, chunk):
        x[t0:t0 + chunk] = (torch.randn(chunk, N_IN, generator=g, device=device) * scale).to(torch.bfloat16)
    return w, x


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = ROOT / "gpurun_out" / f"clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.path.parent.mkdir(exist_ok=True)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        rows = []
        for line in self.path.read_text().splitlines():
            f = [v.strip() for v in line.split(",")]
            if len(f) >= 8:
                rows.append(f)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------- CPU reference arm
def cpu_reference(steps: int, warmup: int, chunk: int = 1024, threads: int | None = None):
    """The reference's own CPU implementation (oracle/_ref: proj/src compiled
    unmodified) on the same config.  Sample: the full-layer gptq_quantize once
    (H precomputed from a chunk), then `steps` accumulate_stats calls on
    `chunk`-token slices; per-layer time = t_gptq + (T/chunk) * mean(t_stats)."""
    from oracle import ocw_oracle as orc
    from oracle import ref
    threads = threads or os.cpu_count() or 1
    os.environ["OCW_SHIM_THREADS"] = str(threads)
    ref.use_blas(True)
    ref.set_threads(threads)
    rng = np.random.default_rng(SEED_W)
    w = orc.bf16_round((rng.standard_normal((N_IN, M_OUT), dtype=np.float32) * 0.02))
    scale = np.ones(N_IN, np.float32)
    scale[outlier_channels(N_IN, 0.01, SEED_PICK)] = 20.0
    gram, cross = np.zeros((N_IN, N_IN)), np.zeros((N_IN, N_IN))
    t_stats = []
    for s in range(warmup + steps):
        x = orc.bf16_round(rng.standard_normal((chunk, N_IN), dtype=np.float32) * scale)
        _, sec = ref.accumulate_stats(gram, cross, x, x, timing=True)
        if s >= warmup:
            t_stats.append(sec)
    h = gram.astype(np.float32)
    _, _, _, t_gptq = ref.gptq_quantize(w, h, BITS, 1, 2, GROUP, True, 0.01, 128, timing=True)
    t_layer = t_gptq + (TOKENS / chunk) * statistics.mean(t_stats)
    return {
        "value": N_IN * M_OUT / t_layer, "unit": "weights/s", "cores": threads, "kind": "reference",
        "t_layer_s": t_layer, "t_gptq_s": t_gptq, "t_stats_chunk_s": statistics.mean(t_stats),
        "blas": ref.blas_name(),
        "sample": (f"reference proj/src (quant/stats/layerwise.cpp) built by oracle/build_ref.sh, "
                   f"OpenBLAS {threads} threads for its fp64 GEMM/LLT; full 4096x4096 gptq_quantize "
                   f"once + {steps} accumulate_stats calls of {chunk} tokens, stats extrapolated "
                   f"x{TOKENS // chunk} to {TOKENS} tokens"),
    }


def cpu_baseline_subprocess(threads: int, steps: int, timeout: float = 600.0):
    """The CPU baseline leg in its own process (the product process never maps
    the oracle library): prints one JSON object."""
    cmd = [sys.executable, str(Path(__file__).resolve()), "--cpu-baseline-only", str(threads),
           "--steps", str(steps)]
    env = dict(os.environ, OMP_NUM_THREADS=str(threads), OPENBLAS_NUM_THREADS=str(threads))
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    if r.returncode != 0 or not lines:
        raise RuntimeError(f"cpu baseline ({threads} threads) failed: {r.stderr[-400:]}")
    return json.loads(lines[-1])


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cb = cpu_reference(args.steps, args.warmup)
    line = {
        "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "weights/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": cb["t_layer_s"] * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C2 llama2-7b q_proj 4096x4096 W4 g128 act-order, 262144 tokens",
                   "orientation": "reference (N=in rows)"},
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": cb["value"], "unit": "weights/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- C4 model sweep
def run_model_mode(args):
    """BASELINE.json configs[3]: the whole 7B-shaped model (32 blocks x 7
    linears, W4 g128, act-order, 262144 tokens per tap), the 128 distinct-input
    units spread over the ranks by LPT; each step is one full sweep (synthetic
    X and W generated on the device, then Hessian / factor / sweeps / pack);
    wall-clock = max over ranks of the device time of the step."""
    import torch
    import torch.distributed as dist

    from paper_2603_28845_b200 import dev
    from paper_2603_28845_b200 import model_sweep as MS

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    device = torch.device("cuda", local)
    units = MS.model_units(args.blocks)
    plan = MS.lpt(units, world)
    mine = plan[rank]
    for _ in range(args.warmup):  # warm: one unit of each shape
        seen, warm = set(), []
        for u in mine:
            if (u.n, u.linears) not in seen:
                seen.add((u.n, u.linears))
                warm.append(u)
        MS.run_rank(warm, local, keep_payload=False)
    clocks = ClockSampler(local)
    l0 = dev.launch_count()
    walls, stats = [], None
    for _ in range(args.steps):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        if not walls:
            clocks.start()
        payloads, stats = MS.run_rank(mine, local, keep_payload=True)
        ms = torch.tensor([stats["ms"], stats["quant_ms"]], device=device)
        if world > 1:
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        walls.append((float(ms[0].item()), float(ms[1].item())))
        del payloads
    ck = clocks.stop()
    launches = dev.launch_count() - l0
    total_w = sum(u.n * m for u in units for _, m in u.linears)
    loads = [sum(MS.unit_cost(u) for u in p) for p in plan]
    if rank == 0:
        wall = statistics.mean(w for w, _ in walls)
        qwall = statistics.mean(q for _, q in walls)
        line = {
            "metric": "C4 whole-model sweep throughput (weights/s), 32 x 7 Llama-2-7B linears W4 g128",
            "value": total_w / (qwall / 1e3), "unit": "weights/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": qwall,
            "quantize_wall_clock_s": qwall / 1e3,
            "wall_clock_s_with_input_generation": wall / 1e3,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16 (Hessian); fp32 factor/sweep", "data": "synthetic",
            "config": {"workload": f"C4: {args.blocks} blocks x 7 linears (q/k/v/o 4096x4096, gate/up "
                                   f"4096x11008, down 11008x4096, reference orientation), "
                                   f"{TOKENS} tokens per tap, 4 distinct taps per block",
                       "parallelism": f"{len(units)} units by LPT over {world} ranks",
                       "lpt_balance": max(loads) / (sum(loads) / world)},
            "rank0": stats, "gpu_launches": launches, "clocks": ck,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-baseline-only", type=int, default=0, metavar="THREADS",
                    help="(internal) run the CPU baseline leg with THREADS threads, print JSON")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-dropin", action="store_true",
                    help="skip the reference-API leg (lib/dropin_bench: ocw::accumulate_stats + "
                         "ocw::quantize_layer on fp32 host matrices)")
    ap.add_argument("--mode", default="layers", choices=["layers", "sharded", "model"],
                    help="N>1: layers = one layer per rank (weak); sharded = one layer split "
                         "over ranks: token-sharded Hessian + NCCL all-reduce + column slabs + "
                         "gather to rank 0 (strong); model = BASELINE configs[3] (C4): the whole "
                         "7B-shaped model sweep, units spread over the ranks by LPT (strong)")
    ap.add_argument("--blocks", type=int, default=32, help="--mode model: decoder blocks")
    args = ap.parse_args()
    if args.cpu_baseline_only:
        cb = cpu_reference(steps=args.steps, warmup=0, chunk=1024, threads=args.cpu_baseline_only)
        print(json.dumps(cb), flush=True)
        return
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.mode == "model":
        return run_model_mode(args)

    import torch
    import torch.distributed as dist

    import paper_2603_28845_b200 as g
    from paper_2603_28845_b200 import dev

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    device = torch.device("cuda", local)

    cfg = g.QuantConfig(BITS, g.Scheme.asymmetric, g.Granularity.per_group, GROUP)
    opts = g.GptqOptions(actorder=True, percdamp=0.01, block_cols=128)
    w, x = make_inputs(device, torch)
    sharded = args.mode == "sharded"
    out = dev.LayerBuffers(N_IN, M_OUT, cfg, local, w_hat=not sharded, payload=not sharded)
    stream = torch.cuda.current_stream(device)
    if sharded:  # this rank's token shard; slabs + gather in paper_2603_28845_b200/dist.py
        from paper_2603_28845_b200 import dist as D
        t0, t1 = D.token_range(TOKENS, rank, world)
        x = x[t0:t1].contiguous()  # (synthetic: every rank draws the same stream, keeps its shard)
        j0, j1 = D.column_slabs(M_OUT, GROUP, BITS, world)[rank] if world > 1 else (0, M_OUT)
        ops = D.gpu_ops(local, w_hat=True)

    def step(ev=None):
        if ev is not None:
            ev[0].record(stream)
        dev.hessian(x, out.h)
        if sharded and world > 1:
            dist.all_reduce(out.h, op=dist.ReduceOp.SUM)  # the one exchange step (NCCL)
        if ev is not None:
            ev[1].record(stream)
        if sharded:
            res = ops.gptq_slab(w, j0, j1, out.h, cfg, opts)  # grids + sweep + pack of the slab
            if ev is not None:
                ev[2].record(stream)
            D.gather_slabs(res, N_IN, M_OUT, GROUP, BITS, True)  # to rank 0 + per-row assembly
        else:
            dev.gptq(w, out.h, cfg, opts, out)
            if ev is not None:
                ev[2].record(stream)
            dev.pack(out, cfg)
        if ev is not None:
            ev[3].record(stream)

    for _ in range(args.warmup):
        step()
    dev.synchronize(local)
    dev.profile(True)
    step()
    phases = dev.profile(False)
    dev.synchronize(local)
    # timed steps: device calls only enqueue (errors latched, raised at synchronize)
    dev.set_async(True, local)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    clocks = ClockSampler(local)
    clocks.start()
    l0 = dev.launch_count()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for k in range(args.steps):
        step(evs[k])
    t_end.record(stream)
    torch.cuda.synchronize()
    dev.synchronize(local)
    dev.set_async(False, local)
    launches = dev.launch_count() - l0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ck = clocks.stop()
    total_ms = t_start.elapsed_time(t_end)
    if world > 1:
        tt = torch.tensor([total_ms], device=device)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    ms_step = total_ms / args.steps
    t_h = statistics.mean(e[0].elapsed_time(e[1]) for e in evs)
    t_q = statistics.mean(e[1].elapsed_time(e[2]) for e in evs)
    t_p = statistics.mean(e[2].elapsed_time(e[3]) for e in evs)
    value = (1 if sharded else world) * N_IN * M_OUT / (ms_step / 1e3)

    # ---- end to end through the public host API (pinned host buffers, H2D + D2H in the region)
    e2e = None
    if args.e2e_steps > 0:
        xh = x.cpu().pin_memory()
        wh = w.cpu().pin_memory()
        xb = xh.view(torch.int16).numpy().view(np.uint16)
        wb = wh.numpy()

        def pinned(shape, dtype):  # host outputs in pinned memory (full-rate D2H)
            nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
            buf = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
            return buf.numpy().view(dtype).reshape(shape)

        # the reference quantize_layer's outputs (codes + grids, layerwise.cpp:120-126)
        # plus the OCW1 payload; W_hat is dequantize(), a separate call
        outs = g.LayerOutputs(N_IN, M_OUT, cfg, alloc=pinned, with_h=False, with_w_hat=False)
        g.quantize_layer_x(wb, xb, cfg, opts, out=outs)  # warm (allocations)
        times = []
        for _ in range(args.e2e_steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            q, payload, _h = g.quantize_layer_x(wb, xb, cfg, opts, out=outs)
            times.append(time.perf_counter() - t0)
        t_e2e = statistics.mean(times)
        h2d = TOKENS * N_IN * 2 + N_IN * M_OUT * 4
        ng = N_IN * (M_OUT // GROUP)
        d2h = N_IN * M_OUT * 2 + ng * 8 + len(payload)
        e2e = {"value": world * N_IN * M_OUT / t_e2e, "unit": "weights/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": t_e2e * 1e3,
               "api": "paper_2603_28845_b200.quantize_layer_x -> ocwg_quantize_layer_x (host buffers: "
                      "W, X in; codes, scales, zeros, payload out -- the reference quantize_layer's result plus the "
                      "OCW1 payload; X streamed in 32768-token "
                      "chunks under the Hessian)"}

    # ---- the reference's own API path through the C++ drop-in (fp32 host matrices,
    # X_hat != X; what run_layerwise_sweep calls per layer, pipeline.cpp:215-226)
    dropin = None
    exe = ROOT / "paper_2603_28845_b200" / "lib" / "dropin_bench"
    if world == 1 and not args.no_dropin and not sharded and exe.exists():
        try:
            torch.cuda.synchronize()
            r = subprocess.run([str(exe), str(TOKENS), str(N_IN), str(M_OUT)], capture_output=True,
                               text=True, timeout=900,
                               env=dict(os.environ, OCWG_DEVICE=str(local)))
            js = [l for l in r.stdout.splitlines() if l.startswith("{")]
            dropin = json.loads(js[-1]) if r.returncode == 0 and js else {"error": r.stderr[-300:]}
            if "layer_ms" in dropin:
                dropin["value"] = N_IN * M_OUT / (dropin["layer_ms"] / 1e3)
                dropin["unit"] = "weights/s"
                dropin["api"] = ("ocw::accumulate_stats(stats, x_fp, x_hat) + ocw::quantize_layer(w, stats, "
                                 "gptq W4 g128 act-order, block_cols 32) through cpp/ocw_dropin.cpp "
                                 "(fp32 host matrices in and out; layer_qep_ms adds QEP alpha 1 eta 0.01)")
        except Exception as e:  # report, never fake
            dropin = {"error": str(e)[:300]}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    peak_burst, peak_sus, peak_bw, peak_src = peaks()
    achieved = F_H / (t_h / 1e3) / 1e12
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        # the reference's CPU path on this box's host cores, in subprocesses:
        # all cores (OpenBLAS threads for Eigen's GEMM/LLT) and 1 core (the
        # reference as built is single-threaded)
        try:
            allc = os.cpu_count() or 1
            cb = cpu_baseline_subprocess(allc, steps=3)
            cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
            try:
                c1 = cpu_baseline_subprocess(1, steps=1)
                cpu["single_core"] = {k: c1[k] for k in ("value", "unit", "cores", "sample")}
            except Exception as e:
                cpu["single_core"] = {"value": None, "sample": f"unavailable: {e}"}
        except Exception as e:  # report, never fake
            cpu = {"value": None, "unit": "weights/s", "cores": None, "kind": "reference",
                   "sample": f"unavailable: {e}"}
    line = {
        "metric": METRIC, "value": value, "unit": "weights/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong" if sharded else "weak",
        "vs_baseline": None,
        "dtype": "bf16 (Hessian, fp32 accumulate); fp32 factor/sweep (3xTF32 tcgen05 GEMMs)",
        "data": "synthetic",
        "config": {"workload": "C2 llama2-7b q_proj: W 4096(in)x4096(out), X 262144x4096 bf16 "
                               "(1% outlier channels x20), W4 asym g128, act-order, damp 0.01, block 128",
                   "l2": "inputs larger than L2 (X = 2 GiB), no flush",
                   "parallelism": (f"one layer over {world} ranks: token-sharded Hessian + NCCL "
                                   f"all-reduce, {GROUP}-aligned column slabs" if sharded else
                                   f"{world} independent layers" if world > 1 else "single GPU")},
        "breakdown_ms": {"hessian": t_h, "gptq": t_q, ("gather" if sharded else "pack"): t_p,
                         "gptq_phases": phases},
        "hessian_tflops": achieved,
        "roofline": {"bound": "tensor", "kernel": "gram_tc_kernel<float>", "achieved": achieved,
                     "peak": peak_burst, "unit": "TFLOP/s", "frac": achieved / peak_burst,
                     "peak_source": f"{peak_src} bf16 burst (MEASURED_PEAKS.json bf16_tflops: the "
                                    f"timed loop is {total_ms / 1e3:.2f} s, short of the seconds-long "
                                    f"sustained measurement); of the sustained {peak_sus}: "
                                    f"frac {achieved / peak_sus:.3f}",
                     "algorithmic": "T*N*(N+1) flops per launch",
                     "traffic": HESSIAN_TRAFFIC_BYTES if not sharded else None,
                     "traffic_source": "ncu dram__bytes_read.sum + dram__bytes_write.sum, one launch "
                                       "at C2 (profiles/r02_gram_ncu_full.txt)"},
        "gpu_launches": launches,
        "clocks": ck,
        "e2e": e2e,
        "dropin": dropin,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
