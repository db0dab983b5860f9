"""Multi-GPU layer quantize: one process per GPU over
torch.distributed (NCCL over NVLink on the GPUs; gloo for the CPU tests of this
host logic).

The path shards two ways, with exactly one exchange step in the compute:
  * Hessian -- token shards: rank r accumulates H_r = X_r^T X_r over its
    contiguous token range on the tensor cores, then ONE all-reduce (sum,
    fp32) gives every rank the same H (stats.cpp:16 is a sum over tokens).
  * Sweep -- output-column slabs: columns are independent given H
    (layerwise.cpp:65-91 updates whole rows of W, column by column
    independently), so rank r quantizes W[:, j0:j1) with no communication.
    Slabs are group-aligned: a per-group grid spans G consecutive columns of
    one row (quant.cpp:158-166), and G*b and M*b are multiples of 8 for the
    BASELINE configs, so every slab's packed bits start on a byte boundary in
    each row of the OCW1 bitstream (container.cpp:129-139).
  The factorisation is replicated (each rank factors the same H).
  * Gather -- each rank flattens its slab results (codes, grids, payload
    bitstream rows, fp16 scales, u8 zeros) into ONE byte buffer on its device;
    a collective gather brings them to rank 0 (NCCL: NVLink P2P), and rank 0
    interleaves them per row into the full layer with strided device copies
    (byte copies; no re-quantisation, no host round trip).

Per-tensor and per-channel grids span all columns of W, so they cannot be
split by columns: those granularities run unsharded (world == 1).
"""
from __future__ import annotations

from dataclasses import dataclass


def token_range(tokens: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced token shard [t0, t1) of rank `rank`."""
    base, extra = divmod(tokens, world)
    t0 = rank * base + min(rank, extra)
    return t0, t0 + base + (1 if rank < extra else 0)


def column_slabs(m: int, group: int, bits: int, world: int) -> list[tuple[int, int]]:
    """Group-aligned, balanced output-column slabs [j0, j1), one per rank."""
    if (group * bits) % 8 or (m * bits) % 8:
        raise ValueError("column slabs need G*b and M*b to be multiples of 8 (byte-aligned rows)")
    ngroups = (m + group - 1) // group
    if world > ngroups:
        raise ValueError(f"{world} ranks but only {ngroups} column groups")
    slabs = []
    for r in range(world):
        g0, g1 = token_range(ngroups, r, world)
        slabs.append((g0 * group, min(m, g1 * group)))
    return slabs


@dataclass
class SlabResult:
    """One rank's quantized slab W[:, j0:j1) as torch tensors (device or CPU):
    codes int16 [N, ms], slab-local grids (row-major over (row, slab group))
    scales fp32 / zeros int32, w_hat fp32 [N, ms] or None, and the slab's own
    OCW1 payload (uint8: bitstream, fp16 scales, u8 zeros)."""
    j0: int
    j1: int
    codes: object
    scales: object
    zeros: object
    w_hat: object
    payload: object


def _layout(n: int, j0: int, j1: int, group: int, bits: int, asym: bool, with_w_hat: bool):
    """Byte offsets of a slab's fields in its flat gather buffer."""
    ms = j1 - j0
    gs = (j1 + group - 1) // group - j0 // group
    sizes = [("codes", n * ms * 2), ("scales", n * gs * 4), ("zeros", n * gs * 4),
             ("payload", n * ms * bits // 8 + n * gs * (3 if asym else 2))]
    if with_w_hat:
        sizes.append(("w_hat", n * ms * 4))
    off, out = 0, {}
    for name, b in sizes:
        out[name] = (off, b)
        off += (b + 15) // 16 * 16
    return out, off


def _flatten(res: SlabResult, layout: dict, total: int, torch):
    buf = torch.zeros(total, dtype=torch.uint8, device=res.codes.device)
    for name, (off, b) in layout.items():
        t = getattr(res, name)
        buf[off:off + b] = t.contiguous().view(-1).view(torch.uint8)
    return buf


def _rank_world(group=None) -> tuple[int, int]:
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def gather_slabs(res: SlabResult, n: int, m: int, group: int, bits: int, asym: bool,
                 group_pg=None):
    """Collective: every rank's slab to rank 0 (one padded byte buffer per
    rank), then the per-row interleave into the full layer on rank 0's device.
    Returns (codes [N, M] int16, scales [N * gpr] fp32, zeros int32, w_hat or
    None, payload uint8) on rank 0, None elsewhere."""
    import torch
    import torch.distributed as dist

    rank, world = _rank_world(group_pg)
    slabs = column_slabs(m, group, bits, world) if world > 1 else [(0, m)]
    with_w_hat = res.w_hat is not None
    layouts = [_layout(n, a, b, group, bits, asym, with_w_hat) for a, b in slabs]
    cap = max(t for _, t in layouts)
    mine = _flatten(res, layouts[rank][0], cap, torch)
    if world > 1:
        parts = [torch.empty(cap, dtype=torch.uint8, device=mine.device) for _ in range(world)] \
            if rank == 0 else None
        dist.gather(mine, parts, dst=0, group=group_pg)
    else:
        parts = [mine]
    if rank != 0:
        return None
    dv = mine.device
    gpr = (m + group - 1) // group
    row_bytes = m * bits // 8
    codes = torch.empty((n, m), dtype=torch.int16, device=dv)
    scales = torch.empty((n, gpr), dtype=torch.float32, device=dv)
    zeros = torch.empty((n, gpr), dtype=torch.int32, device=dv)
    w_hat = torch.empty((n, m), dtype=torch.float32, device=dv) if with_w_hat else None
    cbits = torch.empty((n, row_bytes), dtype=torch.uint8, device=dv)
    sc16 = torch.empty((n, 2 * gpr), dtype=torch.uint8, device=dv)
    z8 = torch.empty((n, gpr), dtype=torch.uint8, device=dv)
    for (j0, j1), (lay, _), buf in zip(slabs, layouts, parts):
        ms = j1 - j0
        g0, g1 = j0 // group, (j1 + group - 1) // group
        gs = g1 - g0

        def field(name, dtype, shape):
            off, b = lay[name]
            return buf[off:off + b].view(dtype).view(*shape)

        codes[:, j0:j1] = field("codes", torch.int16, (n, ms))
        scales[:, g0:g1] = field("scales", torch.float32, (n, gs))
        zeros[:, g0:g1] = field("zeros", torch.int32, (n, gs))
        if with_w_hat:
            w_hat[:, j0:j1] = field("w_hat", torch.float32, (n, ms))
        # the slab payload: its own row-major bitstream, fp16 scales, u8 zeros
        off, _ = lay["payload"]
        srow = ms * bits // 8
        p = buf[off:]
        cbits[:, j0 * bits // 8:j1 * bits // 8] = p[:n * srow].view(n, srow)
        sc16[:, 2 * g0:2 * g1] = p[n * srow:n * srow + 2 * n * gs].view(n, 2 * gs)
        if asym:
            z8[:, g0:g1] = p[n * srow + 2 * n * gs:n * srow + 3 * n * gs].view(n, gs)
    code_bytes = (n * m * bits + 7) // 8
    pieces = [cbits.view(-1)[:code_bytes], sc16.view(-1)] + ([z8.view(-1)] if asym else [])
    payload = torch.cat(pieces)
    return codes, scales.view(-1), zeros.view(-1), w_hat, payload


def quantize_layer_sharded(w, x_local, tokens: int, cfg, opts, group=None, ops=None):
    """Token-sharded Hessian + one all-reduce + column-slab GPTQ + gather;
    rank 0 returns the assembled full result (codes, scales, zeros, w_hat,
    payload) as tensors on its device, the other ranks None.

    `ops` supplies the per-rank compute: ``gram(x_local) -> H_local`` (N x N
    tensor) and ``gptq_slab(w, j0, j1, H) -> SlabResult`` -- the GPU
    implementations by default (``gpu_ops``); tests substitute the CPU oracle
    to check this host logic under gloo.
    """
    import torch.distributed as dist

    ops = ops or gpu_ops()
    rank, world = _rank_world(group)
    n, m = w.shape
    if world > 1 and int(cfg.granularity) != 2:
        raise ValueError("column sharding needs per-group grids (per-tensor/per-channel span all columns)")
    h = ops.gram(x_local)                         # H_r = X_r^T X_r
    if world > 1:
        dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)  # the one exchange step
    group_size = int(cfg.group_size) if int(cfg.granularity) == 2 else m
    slabs = column_slabs(m, group_size, int(cfg.bits), world) if world > 1 else [(0, m)]
    j0, j1 = slabs[rank]
    res = ops.gptq_slab(w, j0, j1, h, cfg, opts)
    return gather_slabs(res, n, m, group_size, int(cfg.bits), int(cfg.scheme) == 1, group)


class gpu_ops:
    """Per-rank compute on this rank's GPU (libocwg.so through dev.py)."""

    def __init__(self, device: int | None = None, w_hat: bool = True):
        import torch
        self.torch = torch
        self.device = torch.cuda.current_device() if device is None else device
        self.w_hat = w_hat
        self.bufs = {}

    def gram(self, x_local):
        from . import dev
        h = self.torch.empty((x_local.shape[1],) * 2, dtype=self.torch.float32,
                             device=f"cuda:{self.device}")
        dev.hessian(x_local, h)
        return h

    def gptq_slab(self, w, j0, j1, h, cfg, opts):
        from . import dev, quant_group_count
        n, m = w.shape
        ms = j1 - j0
        key = (n, ms)
        if key not in self.bufs:  # output buffers reused across calls
            self.bufs[key] = dev.LayerBuffers(n, ms, cfg, self.device, w_hat=self.w_hat, h=False)
        out = self.bufs[key]
        ws = w if (j0 == 0 and j1 == m) else w[:, j0:j1].contiguous()
        dev.gptq(ws, h, cfg, opts, out)
        dev.pack(out, cfg)
        ng = quant_group_count(cfg, n, ms)
        return SlabResult(j0, j1, out.codes, out.scales[:ng], out.zeros[:ng], out.w_hat,
                          out.payload)
