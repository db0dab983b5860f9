"""Per-layer times of the other BASELINE.json configs on one GPU (C3 up/down,
C5 up/down; configs[2], configs[4]) through the device API, with seeded
synthetic inputs of the configs' shapes and distributions (no dataset: see
DESIGN.md).  Not the bench contract's headline (that is C2 in bench.py); a
check that the large shapes run (macro-panel Cholesky for n > 4608, wide
sweeps) and what they cost.  Sanity per layer: codes in range and the
activation-weighted error of GPTQ below RTN's on a token subsample.

    python tools/bench_configs.py [--reps 2] [--only c3up,c3down,c5up,c5down]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2603_28845_b200 as g  # noqa: E402
from paper_2603_28845_b200 import dev  # noqa: E402

T = 262144
CONFIGS = {  # name: (N in, M out, bits, group, outlier frac, outlier scale, W std, silu X)
    "c3up": (4096, 11008, 3, 128, 0.01, 20.0, 0.02, False),
    "c3down": (11008, 4096, 3, 128, 0.0, 1.0, 0.02, True),
    "c5up": (8192, 28672, 2, 64, 0.005, 30.0, 0.015, False),
    "c5down": (28672, 8192, 2, 64, 0.005, 30.0, 0.015, False),
}


def inputs(n, m, frac, osc, wstd, silu, seed):
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    w = (torch.randn(n, m, generator=gen, device="cuda") * wstd).to(torch.bfloat16).float()
    x = torch.empty(T, n, dtype=torch.bfloat16, device="cuda")
    scale = torch.ones(n, device="cuda")
    k = int(round(frac * n))
    if k:
        scale[torch.randperm(n, generator=gen, device="cuda")[:k]] = osc
    chunk = 8192
    for t0 in range(0, T, chunk):
        if silu:
            a = torch.randn(chunk, n, generator=gen, device="cuda")
            b = torch.randn(chunk, n, generator=gen, device="cuda")
            x[t0:t0 + chunk] = (torch.nn.functional.silu(a) * b).to(torch.bfloat16)
        else:
            x[t0:t0 + chunk] = (torch.randn(chunk, n, generator=gen, device="cuda") * scale).to(torch.bfloat16)
    return w, x


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--only", default="c3up,c3down,c5up,c5down")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    out = {}
    for name in args.only.split(","):
        n, m, bits, grp, frac, osc, wstd, silu = CONFIGS[name]
        w, x = inputs(n, m, frac, osc, wstd, silu, 1234 + n + m)
        cfg = g.QuantConfig(bits, g.Scheme.asymmetric, g.Granularity.per_group, grp)
        opts = g.GptqOptions(actorder=True, percdamp=0.01, block_cols=128)
        buf = dev.LayerBuffers(n, m, cfg, 0)
        times = []
        for rep in range(args.reps + 1):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dev.hessian(x, buf.h)
            dev.gptq(w, buf.h, cfg, opts, buf)
            dev.pack(buf, cfg)
            torch.cuda.synchronize()
            if rep:
                times.append(time.perf_counter() - t0)
        codes = buf.codes
        qmax = (1 << bits) - 1
        ok_range = bool((codes.min() >= 0).item() and (codes.max() <= qmax).item())
        # activation-weighted error on a token subsample, GPTQ vs RTN
        xs = x[:8192].float()
        rtn_codes = torch.empty_like(buf.codes)
        q_rtn = g.quantize_matrix(w.cpu().numpy(), cfg)
        wr = torch.from_numpy(g.dequantize(q_rtn)).cuda()
        err_g = torch.linalg.norm(xs @ (buf.w_hat - w)).item()
        err_r = torch.linalg.norm(xs @ (wr - w)).item()
        del rtn_codes
        out[name] = {"n": n, "m": m, "bits": bits, "group": grp, "tokens": T,
                     "ms_per_layer": 1e3 * float(np.mean(times)),
                     "weights_per_s": n * m / float(np.mean(times)),
                     "codes_in_range": ok_range, "act_err_gptq_over_rtn": err_g / err_r}
        print(json.dumps({name: out[name]}), flush=True)
        del w, x, buf, xs, wr
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
