"""Time the JointQ refiner on the GPU against the reference's own
jointq.cpp (oracle/_ref, CPU) on a GPTQ-initialised layer.

    python tools/jointq_bench.py [--c2-tokens T] [--skip-cpu]

C1: BASELINE configs[0] shapes (W 512 x 512 ~N(0, 0.02^2), X 4096 x 512 bf16-valued
N(0,1), W4 asymmetric g128; GPTQ start without act-order, damp 0.01), lambda 0.2,
8 passes, radius 1 -- both implementations, results compared.
C2: the 4096 x 4096 W4 g128 layer (X: T x 4096; the search cost does not depend on
T) -- GPU only (the CPU reference needs tens of minutes per pass there).
Prints one JSON line per case."""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2603_28845_b200 as g  # noqa: E402
from oracle import ocw_oracle as orc  # noqa: E402
from oracle import ref  # noqa: E402


def layer(n, m, tokens, seed):
    w = ref.random_gaussian(n, m, seed, 0.02)
    x = orc.bf16_round(ref.random_gaussian(tokens, n, seed + 1))
    cfg = g.QuantConfig(4, g.Scheme.asymmetric, g.Granularity.per_group, 128)
    if n > 1024:  # the GPTQ start's H on the device (numpy fp64 would take minutes)
        import torch
        xt = torch.from_numpy(x).cuda().double()
        h = (xt.T @ xt).float().cpu().numpy()
    else:
        h = (x.T.astype(np.float64) @ x.astype(np.float64)).astype(np.float32)
    q = g.gptq_quantize(w, h, cfg, g.GptqOptions(False, 0.01, 128))
    return w, x, q


def run(name, n, m, tokens, cpu):
    w, x, q0 = layer(n, m, tokens, 0x7A11 + n)
    opts = g.JointqOptions(0.2, 8, 1)
    wq, xq, qq = layer(64, 128, 256, 3)  # warm-up (context, module load)
    g.jointq_refine(qq, wq, xq, opts)
    t0 = time.perf_counter()
    res = g.jointq_refine(q0, w, x, opts)
    t_gpu = time.perf_counter() - t0
    out = {"case": name, "n": n, "m": m, "tokens": tokens, "config": "W4 asym g128, GPTQ start",
           "lambda": 0.2, "passes": res.passes, "accepted_moves": res.accepted_moves,
           "J0": float(res.objective_trace[0]), "J": float(res.objective_trace[-1]),
           "gpu_s": round(t_gpu, 4),
           "api": "paper_2603_28845_b200.jointq_refine -> ocwg_jointq_refine (host buffers; "
                  "includes X / W transfer, H = X^T X and G = H E setup)"}
    if cpu:
        ref.lib().ocwref_use_blas(1)
        t0 = time.perf_counter()
        rc, rs, rz, rtrace, racc, rpass = ref.jointq_refine(q0.codes, q0.scales, q0.zeros, w, x, 4, 1,
                                                            2, 128, 0.2, 8, 1)
        t_cpu = time.perf_counter() - t0
        out.update({"cpu_s": round(t_cpu, 3), "cpu_impl": "reference jointq.cpp (oracle/_ref), "
                    "1 thread for the search, OpenBLAS for its two GEMMs",
                    "cpu_accepted_moves": racc, "cpu_passes": rpass, "cpu_J": float(rtrace[-1]),
                    "codes_identical": float(np.mean(res.refined.codes == rc)),
                    "scales_identical": bool(np.array_equal(res.refined.scales, rs)),
                    "speedup": round(t_cpu / t_gpu, 1)})
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c2-tokens", type=int, default=16384)
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-c2", action="store_true")
    a = ap.parse_args()
    run("C1", 512, 512, 4096, not a.skip_cpu)
    if not a.skip_c2:
        run("C2", 4096, 4096, a.c2_tokens, False)


if __name__ == "__main__":
    main()
