"""One C2 layer (BASELINE.json configs[1]) through the device API, for ncu.

Generates the bench inputs, runs `--reps` full steps (Hessian -> factorise ->
sweep -> pack) and exits.  Used as the plain run and the ncu target:
  python tools/prof_c2.py --reps 2
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_28845_b200 as g  # noqa: E402
from paper_2603_28845_b200 import dev  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    cfg = g.QuantConfig(bench.BITS, g.Scheme.asymmetric, g.Granularity.per_group, bench.GROUP)
    opts = g.GptqOptions(actorder=True, percdamp=0.01, block_cols=128)
    w, x = bench.make_inputs(torch.device("cuda", 0), torch)
    out = dev.LayerBuffers(bench.N_IN, bench.M_OUT, cfg, 0)
    torch.cuda.synchronize()
    for _ in range(args.reps):
        dev.hessian(x, out.h)
        dev.gptq(w, out.h, cfg, opts, out)
        dev.pack(out, cfg)
    torch.cuda.synchronize()
    print("prof_c2 ok", dev.launch_count())


if __name__ == "__main__":
    main()
