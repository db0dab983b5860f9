"""Multi-GPU layer quantize: one process per GPU over
torch.distributed (NCCL on the GPUs; gloo for the CPU tests of this host logic).

The path shards two ways, with exactly one exchange step:
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
  * Assembly -- rank 0 gathers the slab results and interleaves them per row
    into the full codes / grids / payload (byte copies; no re-quantisation).

Per-tensor and per-channel grids span all columns of W, so they cannot be
split by columns: those granularities run unsharded (world == 1).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


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
    """One rank's quantized slab W[:, j0:j1): codes N x ms, slab-local grids
    (row-major over (row, slab group)), W_hat N x ms, slab OCW1 payload."""
    j0: int
    j1: int
    codes: np.ndarray
    scales: np.ndarray
    zeros: np.ndarray
    w_hat: np.ndarray | None
    payload: bytes


def assemble(slabs: list[SlabResult], n: int, m: int, group: int, bits: int, asym: bool):
    """Interleave slab results per row into the full (codes, scales, zeros,
    w_hat, payload) of the N x M layer -- byte copies only."""
    gpr = (m + group - 1) // group
    codes = np.empty((n, m), np.int16)
    scales = np.empty((n, gpr), np.float32)
    zeros = np.empty((n, gpr), np.int32)
    w_hat = None if slabs[0].w_hat is None else np.empty((n, m), np.float32)
    code_bytes = (n * m * bits + 7) // 8
    row_bytes = m * bits // 8
    cbits = np.empty((n, row_bytes), np.uint8)
    sc16 = np.empty((n, gpr), "<u2")
    z8 = np.empty((n, gpr), np.uint8)
    for s in slabs:
        ms = s.j1 - s.j0
        g0, g1 = s.j0 // group, (s.j1 + group - 1) // group
        codes[:, s.j0:s.j1] = s.codes.reshape(n, ms)
        scales[:, g0:g1] = s.scales.reshape(n, g1 - g0)
        zeros[:, g0:g1] = s.zeros.reshape(n, g1 - g0)
        if w_hat is not None:
            w_hat[:, s.j0:s.j1] = s.w_hat.reshape(n, ms)
        # the slab payload: its own row-major bitstream, fp16 scales, u8 zeros
        p = np.frombuffer(s.payload, np.uint8)
        srow = ms * bits // 8
        sng = n * (g1 - g0)
        cbits[:, s.j0 * bits // 8:s.j1 * bits // 8] = p[:n * srow].reshape(n, srow)
        sc16[:, g0:g1] = p[n * srow:n * srow + 2 * sng].view("<u2").reshape(n, g1 - g0)
        if asym:
            z8[:, g0:g1] = p[n * srow + 2 * sng:n * srow + 3 * sng].reshape(n, g1 - g0)
    payload = cbits.tobytes()[:code_bytes] + sc16.tobytes() + (z8.tobytes() if asym else b"")
    return codes, scales.ravel(), zeros.ravel(), w_hat, payload


def quantize_layer_sharded(w, x_local, tokens: int, cfg, opts, group=None, ops=None):
    """Token-sharded Hessian + one all-reduce + column-slab GPTQ; rank 0
    returns the assembled full result (codes, scales, zeros, w_hat, payload),
    the other ranks None.

    `ops` supplies the per-rank compute: ``gram(x_local) -> H_local`` (fp32
    N x N) and ``gptq_slab(w_slab, H) -> SlabResult-like tuple`` -- the GPU
    implementations by default (``gpu_ops``); tests substitute the CPU oracle
    to check this host logic under gloo.
    """
    import torch
    import torch.distributed as dist

    ops = ops or gpu_ops()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    n, m = w.shape
    if world > 1 and int(cfg.granularity) != 2:
        raise ValueError("column sharding needs per-group grids (per-tensor/per-channel span all columns)")
    h = ops.gram(x_local)                         # H_r = X_r^T X_r
    ht = ops.as_tensor(h)
    if world > 1:
        dist.all_reduce(ht, op=dist.ReduceOp.SUM, group=group)  # the one exchange step
    group_size = int(cfg.group_size) if int(cfg.granularity) == 2 else m
    slabs = column_slabs(m, group_size, int(cfg.bits), world)
    j0, j1 = slabs[rank]
    res = ops.gptq_slab(w, j0, j1, ht, cfg, opts)
    gathered = [None] * world
    if world > 1:
        dist.all_gather_object(gathered, res, group=group)
    else:
        gathered = [res]
    if rank != 0:
        return None
    return assemble(gathered, n, m, group_size, int(cfg.bits), int(cfg.scheme) == 1)


class gpu_ops:
    """Per-rank compute on this rank's GPU (libocwg.so through dev.py)."""

    def __init__(self, device: int | None = None):
        import torch
        self.torch = torch
        self.device = torch.cuda.current_device() if device is None else device

    def as_tensor(self, h):
        return h

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
        out = dev.LayerBuffers(n, ms, cfg, self.device)
        dev.gptq(w[:, j0:j1].contiguous(), h, cfg, opts, out)
        dev.pack(out, cfg)
        self.torch.cuda.synchronize(self.device)
        ng = quant_group_count(cfg, n, ms)
        return SlabResult(j0, j1, out.codes.cpu().numpy(), out.scales[:ng].cpu().numpy(),
                          out.zeros[:ng].cpu().numpy(), out.w_hat.cpu().numpy(),
                          out.payload.cpu().numpy().tobytes())
