"""Device-resident entry points (inputs already in HBM), for the sharded /
multi-GPU driver and the benchmark.  Tensors are torch CUDA tensors used
purely as device memory + stream plumbing; all compute is libocwg.so.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import (GptqOptions, QuantConfig, ScaleMode, _check, context, lib, quant_group_count,
               uniform_storage_bytes)


def _bind_stream(device: int):
    """Run on torch's current stream (handle 0 = the legacy default stream)."""
    ctx = context(device)
    _check(lib().ocwg_set_stream(ctx.handle, C.c_void_p(torch.cuda.current_stream(device).cuda_stream)))
    return ctx


def set_async(on: bool, device: int = 0) -> None:
    """Device calls return once enqueued; errors surface at synchronize()."""
    _check(lib().ocwg_set_async(context(device).handle, int(on)))


def synchronize(device: int = 0) -> None:
    """Drain the context's stream and raise any latched device-side error."""
    _check(lib().ocwg_synchronize(context(device).handle))


class LayerBuffers:
    """Output buffers of one layer quantize, allocated once (N x M)."""

    def __init__(self, n: int, m: int, cfg: QuantConfig, device: int, w_hat: bool = True,
                 payload: bool = True, h: bool = True):
        dev = torch.device("cuda", device)
        ng = quant_group_count(cfg, n, m)
        self.codes = torch.empty((n, m), dtype=torch.int16, device=dev)
        self.scales = torch.empty(ng, dtype=torch.float32, device=dev)
        self.zeros = torch.empty(ng, dtype=torch.int32, device=dev)
        self.w_hat = torch.empty((n, m), dtype=torch.float32, device=dev) if w_hat else None
        self.payload_bytes = uniform_storage_bytes(cfg, n, m)
        self.payload = torch.empty(self.payload_bytes, dtype=torch.uint8, device=dev) if payload else None
        self.h = torch.empty((n, n), dtype=torch.float32, device=dev) if h else None


def _p(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def hessian(x_bf16: torch.Tensor, h: torch.Tensor, accumulate: bool = False) -> None:
    """H (+)= X^T X on the tensor cores (tcgen05)."""
    t, n = x_bf16.shape
    ctx = _bind_stream(x_bf16.device.index)
    _check(lib().ocwg_hessian_bf16_dev(ctx.handle, _p(x_bf16), t, n, _p(h), int(accumulate)))


def gptq(w: torch.Tensor, h: torch.Tensor, cfg: QuantConfig, opts: GptqOptions, out: LayerBuffers,
         mode: ScaleMode = ScaleMode.minmax) -> None:
    """GPTQ of a device-resident W (N x M, contiguous) into `out` (N x M)."""
    n, m = w.shape
    if not w.is_contiguous() or tuple(out.codes.shape) != (n, m):
        raise ValueError("gptq: W must be contiguous and match the output buffers")
    ctx = _bind_stream(w.device.index)
    c, o = cfg._c(), opts._c()
    _check(lib().ocwg_gptq_quantize_dev(ctx.handle, _p(w), m, _p(h), n, m, C.byref(c), C.byref(o),
                                        int(mode), _p(out.codes), _p(out.scales), _p(out.zeros),
                                        _p(out.w_hat)))


def pack(out: LayerBuffers, cfg: QuantConfig) -> None:
    n, m = out.codes.shape
    ctx = _bind_stream(out.codes.device.index)
    c = cfg._c()
    _check(lib().ocwg_pack_uniform_dev(ctx.handle, _p(out.codes), _p(out.scales), _p(out.zeros), n, m,
                                       C.byref(c), _p(out.payload)))


def quantize_layer_x(w: torch.Tensor, x_bf16: torch.Tensor, cfg: QuantConfig, opts: GptqOptions,
                     out: LayerBuffers, mode: ScaleMode = ScaleMode.minmax) -> None:
    """One call: Hessian -> factorisation -> GPTQ sweep -> pack, all on device."""
    n, m = w.shape
    ctx = _bind_stream(w.device.index)
    c, o = cfg._c(), opts._c()
    _check(lib().ocwg_quantize_layer_x_dev(ctx.handle, _p(w), _p(x_bf16), x_bf16.shape[0], n, m,
                                           C.byref(c), C.byref(o), int(mode), _p(out.codes),
                                           _p(out.scales), _p(out.zeros), _p(out.w_hat),
                                           _p(out.payload), _p(out.h)))


def quantize_layers(ws: list, x_bf16: torch.Tensor, cfg: QuantConfig, opts: GptqOptions,
                    outs: list, mode: ScaleMode = ScaleMode.minmax) -> None:
    """Layers sharing one calibration input (q/k/v, gate/up): one Hessian and
    one factorisation on the device, then grids + sweep + pack per W."""
    k = len(ws)
    n = ws[0].shape[0]
    ctx = _bind_stream(x_bf16.device.index)
    arr = lambda vals, t: (t * k)(*vals)  # noqa: E731
    wp = arr([w.data_ptr() for w in ws], C.c_void_p)
    mp = arr([w.shape[1] for w in ws], C.c_uint64)
    cp = arr([o.codes.data_ptr() for o in outs], C.c_void_p)
    sp = arr([o.scales.data_ptr() for o in outs], C.c_void_p)
    zp = arr([o.zeros.data_ptr() for o in outs], C.c_void_p)
    pp = arr([o.payload.data_ptr() if o.payload is not None else 0 for o in outs], C.c_void_p)
    c, o = cfg._c(), opts._c()
    _check(lib().ocwg_quantize_layers_x_dev(ctx.handle, k, C.cast(wp, C.c_void_p), C.cast(mp, C.c_void_p),
                                            _p(x_bf16), x_bf16.shape[0], n, C.byref(c), C.byref(o),
                                            int(mode), C.cast(cp, C.c_void_p), C.cast(sp, C.c_void_p),
                                            C.cast(zp, C.c_void_p), C.cast(pp, C.c_void_p)))


def synth(kind: int, seed: int, out: torch.Tensor, stddev: float = 1.0,
          col_scale: torch.Tensor | None = None) -> None:
    """Seeded synthetic inputs on the device (ocwg_synth_dev): kind 0 bf16
    X = g * col_scale, 1 bf16 X = silu(a) * b, 2 fp32 bf16-valued W = g * stddev."""
    rows, cols = out.shape
    ctx = _bind_stream(out.device.index)
    _check(lib().ocwg_synth_dev(ctx.handle, int(kind), int(seed) & ((1 << 64) - 1), rows, cols,
                                float(stddev), _p(col_scale), _p(out)))


def profile(on: bool, device: int = 0):
    """Enable gptq phase events; returns the last run's phase times (ms)."""
    import numpy as np
    out = np.zeros(5, np.float64)
    _check(lib().ocwg_debug_profile(context(device).handle, int(on), C.c_void_p(out.ctypes.data)))
    return dict(zip(["order_damp_build", "cholesky", "inverse", "grids", "sweep"], out.tolist()))


def launch_count() -> int:
    return int(lib().ocwg_launch_count(None))
