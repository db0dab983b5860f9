"""Experiment: the C2 GPTQ phase (order -> Cholesky -> grids -> sweep) replayed
as one CUDA graph against direct stream launches.
    python tools/graph_exp.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_28845_b200 as g  # noqa: E402
from paper_2603_28845_b200 import dev  # noqa: E402

torch.cuda.set_device(0)
cfg = g.QuantConfig(bench.BITS, g.Scheme.asymmetric, g.Granularity.per_group, bench.GROUP)
opts = g.GptqOptions(actorder=True, percdamp=0.01, block_cols=128)
w, x = bench.make_inputs(torch.device("cuda", 0), torch)
out = dev.LayerBuffers(bench.N_IN, bench.M_OUT, cfg, 0)
dev.hessian(x, out.h)
torch.cuda.synchronize()
dev.set_async(True)
for _ in range(3):
    dev.gptq(w, out.h, cfg, opts, out)
dev.synchronize()
ref_codes = out.codes.clone()


def timeit(fn, reps=20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


ms_direct = timeit(lambda: dev.gptq(w, out.h, cfg, opts, out))
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
graph = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    dev.gptq(w, out.h, cfg, opts, out)  # warm on the side stream
    torch.cuda.synchronize()
    with torch.cuda.graph(graph, stream=s):
        dev.gptq(w, out.h, cfg, opts, out)
torch.cuda.synchronize()
out.codes.zero_()
graph.replay()
torch.cuda.synchronize()
same = bool(torch.equal(out.codes, ref_codes))
ms_graph = timeit(graph.replay)
ms_direct2 = timeit(lambda: dev.gptq(w, out.h, cfg, opts, out))
print(f"gptq phase: direct {ms_direct:.4f} / {ms_direct2:.4f} ms, graph replay {ms_graph:.4f} ms, codes identical {same}")
