"""tcgen05 Hessian (pair kernel by default) vs an fp64 reference: symmetry,
relative error (|dH| / sqrt(Hii Hjj)), accumulate mode, and kernel time."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2603_28845_b200 as g
from paper_2603_28845_b200 import dev

dev._bind_stream(0)
for dim, tok, acc in [(512, 65536, 0), (1000, 20000, 0), (4096, 262144, 0), (2048, 131072, 1)]:
    torch.manual_seed(dim)
    x = torch.randn(tok, dim, device="cuda").to(torch.bfloat16)
    ref = torch.zeros(dim, dim, device="cuda", dtype=torch.float64)
    for t0 in range(0, tok, 16384):
        xc = x[t0:t0 + 16384].double()
        ref += xc.T @ xc
    h = torch.zeros(dim, dim, device="cuda")
    if acc:
        h += 3.0
        ref += 3.0
    dev.hessian(x, h, accumulate=bool(acc))
    torch.cuda.synchronize()
    d = torch.sqrt(torch.outer(torch.diag(ref), torch.diag(ref)))
    err = float(((h.double() - ref).abs() / d).max())
    asym = int((h != h.T).sum())
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(3):
        dev.hessian(x, h)
    ev[1].record()
    torch.cuda.synchronize()
    print(f"dim {dim} tok {tok} acc {acc}: max rel err {err:.2e} asym {asym} "
          f"time {ev[0].elapsed_time(ev[1]) / 3:.3f} ms", flush=True)
