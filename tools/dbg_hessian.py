"""Debug: tcgen05 Hessian repeated calls; which calls leave H untouched."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2603_28845_b200 as g

lib = g.lib()
from paper_2603_28845_b200 import dev
dev._bind_stream(0)
cases = [(512, 65536), (512, 65536), (4096, 262144), (4096, 262144), (512, 65536), (2048, 131072),
         (4096, 262080), (4096, 262144)]
for dim, tok in cases:
    torch.manual_seed(0)
    x = torch.randn(tok, dim, device="cuda").to(torch.bfloat16)
    h = torch.full((dim, dim), -7.0, device="cuda")
    rc = lib.ocwg_debug_hessian_dev(g.context().handle, x.data_ptr(), tok, dim, h.data_ptr(), 0, 0)
    torch.cuda.synchronize()
    diag = torch.diag(h)
    ref = (x.float() ** 2).sum(0)
    print(dim, tok, "rc", rc, "untouched", int((h == -7.0).sum()), "diag relerr",
          float(((diag - ref).abs() / ref).max()), flush=True)
