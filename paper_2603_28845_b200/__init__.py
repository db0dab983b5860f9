"""B200-native GPTQ layer-quantize hot path of OneComp (arXiv 2603.28845).

Python host mirror of the reference's ``ocw::`` quantizer interface
(/root/reference/proj/include/ocw/{quant,stats,layerwise}.hpp), bound with
ctypes to the C ABI of ``lib/libocwg.so`` (``include/ocwg.h``).  Same names,
same argument meaning, same error classes as the reference:

    ocw::calibrate_grids   -> calibrate_grids        (quant.cpp:168-196)
    ocw::quantize_matrix   -> quantize_matrix        (quant.cpp:198-210)
    ocw::dequantize        -> dequantize             (quant.cpp:212-218)
    ocw::activation_objective -> activation_objective (quant.cpp:230-236)
    ocw::accumulate_stats  -> accumulate_stats       (stats.cpp:10-19)
    ocw::gptq_order        -> gptq_order             (layerwise.cpp:11-18)
    ocw::gptq_quantize     -> gptq_quantize          (layerwise.cpp:20-93)
    ocw::quantize_layer    -> quantize_layer         (layerwise.cpp:120-126)
    tensor_payload (uniform) -> pack_uniform / unpack_uniform (container.cpp:129-139,168-199)

plus the north_star's one-call ``quantize_layer_x`` (W + calibration tokens X).

Orientation is the reference's: W is N x M (N = input rows), H is N x N.
Every compute call runs CUDA kernels; there is no CPU fallback -- importing
works without a GPU (for the ABI checks), but compute raises ``CudaError``.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from enum import IntEnum
from pathlib import Path

import numpy as np

__all__ = [
    "Scheme", "Granularity", "ScaleMode", "QuantConfig", "GptqOptions", "QuantizedMatrix",
    "CalibStats", "LayerQuantOptions", "QepOptions", "qep_target", "base_method_from_name", "InvalidInput", "NumericError", "IoError", "CudaError",
    "calibrate_grids", "quantize_matrix", "dequantize", "activation_objective",
    "accumulate_stats", "hessian_bf16", "gptq_order", "gptq_quantize", "gptq_factor",
    "quantize_layer", "quantize_layer_x", "LayerOutputs", "pack_uniform", "unpack_uniform",
    "uniform_storage_bytes", "storage_bytes", "quant_group_count", "lib", "context",
]

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("OCWG_LIB", _HERE / "lib" / "libocwg.so"))


# ------------------------------------------------------------------ errors (errors.hpp:9-21)
class InvalidInput(ValueError):
    """ocw::invalid_input."""


class IoError(IOError):
    """ocw::io_error."""


class NumericError(RuntimeError):
    """ocw::numeric_error."""


class CudaError(RuntimeError):
    """CUDA failure, or no usable GPU (there is no CPU fallback)."""


class Unsupported(RuntimeError):
    """Feature not built on the GPU path yet."""


_ERRORS = {1: InvalidInput, 2: IoError, 3: NumericError, 16: CudaError, 17: Unsupported}


# ------------------------------------------------------------------ config types (quant.hpp:12-63)
class Scheme(IntEnum):
    symmetric = 0
    asymmetric = 1


class Granularity(IntEnum):
    per_tensor = 0
    per_channel = 1
    per_group = 2


class ScaleMode(IntEnum):
    minmax = 0
    mse_grid = 1


@dataclass
class QuantConfig:
    bits: int = 4
    scheme: Scheme = Scheme.symmetric
    granularity: Granularity = Granularity.per_group
    group_size: int = 128

    def _c(self) -> "_QCfg":
        return _QCfg(int(self.bits), int(self.scheme), int(self.granularity), 0, int(self.group_size))


@dataclass
class GptqOptions:
    """layerwise.hpp:11-15 (reference default block_cols = 32)."""
    actorder: bool = False
    percdamp: float = 0.01
    block_cols: int = 32

    def _c(self) -> "_GOpt":
        return _GOpt(int(bool(self.actorder)), 0, float(self.percdamp), int(self.block_cols))


@dataclass
class QuantizedMatrix:
    """quant.hpp:54-63; grids as structure-of-arrays (scales fp32, zeros int32)."""
    rows: int
    cols: int
    config: QuantConfig
    codes: np.ndarray            # int16 [rows, cols]
    scales: np.ndarray           # float32 [groups]
    zeros: np.ndarray            # int32 [groups]
    w_hat: np.ndarray | None = None

    @property
    def qmin(self) -> int:
        return 0 if self.config.scheme == Scheme.asymmetric else -((1 << (self.config.bits - 1)) - 1)

    @property
    def qmax(self) -> int:
        b = self.config.bits
        return (1 << b) - 1 if self.config.scheme == Scheme.asymmetric else (1 << (b - 1)) - 1

    def group_count(self) -> int:
        return quant_group_count(self.config, self.rows, self.cols)


@dataclass
class CalibStats:
    """stats.hpp:13-27: fp64 gram / cross, streaming token count."""
    gram: np.ndarray
    cross: np.ndarray
    token_count: int = 0

    @staticmethod
    def zeros(dim: int) -> "CalibStats":
        return CalibStats(np.zeros((dim, dim)), np.zeros((dim, dim)), 0)

    def dim(self) -> int:
        return self.gram.shape[0]

    def gram_matrix(self) -> np.ndarray:
        """stats.cpp:7: fp64 -> fp32."""
        return self.gram.astype(np.float32)


@dataclass
class QepOptions:
    """layerwise.hpp:28-31: propagation strength alpha in [0,1]; lambda = eta * mean(diag(gram))."""
    alpha: float = 1.0
    eta: float = 0.01


@dataclass
class LayerQuantOptions:
    """layerwise.hpp:41-47; qep: QepOptions or None (enabled when set)."""
    method: str = "gptq"
    config: QuantConfig = field(default_factory=QuantConfig)
    scale_mode: ScaleMode = ScaleMode.minmax
    gptq: GptqOptions = field(default_factory=GptqOptions)
    qep: object | None = None


# ------------------------------------------------------------------ ctypes plumbing
class _QCfg(C.Structure):
    _fields_ = [("bits", C.c_int32), ("scheme", C.c_int32), ("granularity", C.c_int32),
                ("reserved", C.c_int32), ("group_size", C.c_uint64)]


class _GOpt(C.Structure):
    _fields_ = [("actorder", C.c_int32), ("reserved", C.c_int32), ("percdamp", C.c_double),
                ("block_cols", C.c_uint64)]


_P = C.c_void_p
_U64 = C.c_uint64
_SIGS = {
    "ocwg_last_error": (C.c_char_p, []),
    "ocwg_version": (C.c_int, []),
    "ocwg_create": (C.c_int, [C.c_int, C.POINTER(_P)]),
    "ocwg_destroy": (C.c_int, [_P]),
    "ocwg_set_stream": (C.c_int, [_P, _P]),
    "ocwg_set_precision": (C.c_int, [_P, C.c_int]),
    "ocwg_set_stats_layout": (C.c_int, [_P, C.c_int]),
    "ocwg_synchronize": (C.c_int, [_P]),
    "ocwg_set_async": (C.c_int, [_P, C.c_int]),
    "ocwg_debug_factor_bench": (C.c_int, [_P, C.c_int, _P, _P]),
    "ocwg_debug_sweep_trace": (C.c_int, [_P, _P, C.c_int]),
    "ocwg_qep_target": (C.c_int, [_P, _P, _P, _P, _U64, _U64, C.c_double, C.c_double, _P]),
    "ocwg_validate_config": (C.c_int, [C.POINTER(_QCfg)]),
    "ocwg_group_count": (_U64, [C.POINTER(_QCfg), _U64, _U64]),
    "ocwg_storage_bytes": (_U64, [C.POINTER(_QCfg), _U64, _U64]),
    "ocwg_calibrate_grids": (C.c_int, [_P, _P, _U64, _U64, C.POINTER(_QCfg), C.c_int, _P, _P]),
    "ocwg_quantize_matrix": (C.c_int, [_P, _P, _U64, _U64, C.POINTER(_QCfg), C.c_int, _P, _P, _P]),
    "ocwg_dequantize": (C.c_int, [_P, _P, _P, _P, _U64, _U64, C.POINTER(_QCfg), _P]),
    "ocwg_activation_objective": (C.c_int, [_P, _P, _P, _P, _U64, _U64, _P]),
    "ocwg_pack_uniform": (C.c_int, [_P, _P, _P, _P, _U64, _U64, C.POINTER(_QCfg), _P, _U64]),
    "ocwg_unpack_uniform": (C.c_int, [_P, _P, _U64, _U64, _U64, C.POINTER(_QCfg), _P, _P, _P]),
    "ocwg_accumulate_stats": (C.c_int, [_P, _P, _P, _U64, _U64, _P, _P, _P]),
    "ocwg_hessian_bf16": (C.c_int, [_P, _P, _U64, _U64, _P, C.c_int]),
    "ocwg_gptq_order": (C.c_int, [_P, _P, _U64, C.c_int, _P]),
    "ocwg_gptq_quantize": (C.c_int, [_P, _P, _P, _U64, _U64, C.POINTER(_QCfg), C.POINTER(_GOpt),
                                     C.c_int, _P, _P, _P, _P]),
    "ocwg_gptq_factor": (C.c_int, [_P, _P, _U64, C.c_int, C.c_double, _P, _P, _P, _P]),
    "ocwg_quantize_layer": (C.c_int, [_P, _P, _P, _P, _U64, _U64, C.c_int, C.POINTER(_QCfg),
                                      C.POINTER(_GOpt), C.c_int, _P, _P, _P, _P, _P]),
    "ocwg_quantize_layer_x": (C.c_int, [_P, _P, _P, _U64, _U64, _U64, C.POINTER(_QCfg),
                                        C.POINTER(_GOpt), C.c_int, _P, _P, _P, _P, _P, _U64, _P]),
    "ocwg_candidate_grid": (C.c_int, [_P, _P, _U64, _U64, C.c_int, _P, _P, _P]),
    "ocwg_quantize_layers_x": (C.c_int, [_P, C.c_int, _P, _P, _P, _U64, _U64, C.POINTER(_QCfg),
                                         C.POINTER(_GOpt), C.c_int, _P, _P, _P, _P, _P]),
    "ocwg_quantize_layer_x_dev": (C.c_int, [_P, _P, _P, _U64, _U64, _U64, C.POINTER(_QCfg),
                                            C.POINTER(_GOpt), C.c_int, _P, _P, _P, _P, _P, _P]),
    "ocwg_hessian_bf16_dev": (C.c_int, [_P, _P, _U64, _U64, _P, C.c_int]),
    "ocwg_quantize_layers_x_dev": (C.c_int, [_P, C.c_int, _P, _P, _P, _U64, _U64, C.POINTER(_QCfg),
                                             C.POINTER(_GOpt), C.c_int, _P, _P, _P, _P]),
    "ocwg_synth_dev": (C.c_int, [_P, C.c_int, _U64, _U64, _U64, C.c_double, _P, _P]),
    "ocwg_gptq_quantize_dev": (C.c_int, [_P, _P, _U64, _P, _U64, _U64, C.POINTER(_QCfg),
                                         C.POINTER(_GOpt), C.c_int, _P, _P, _P, _P]),
    "ocwg_pack_uniform_dev": (C.c_int, [_P, _P, _P, _P, _U64, _U64, C.POINTER(_QCfg), _P]),
    "ocwg_debug_hessian_dev": (C.c_int, [_P, _P, _U64, _U64, _P, C.c_int, C.c_int]),
    "ocwg_debug_split_dev": (C.c_int, [_P, _P, _P, _U64, _U64, _U64, _P, _P, _P, _P, _P]),
    "ocwg_debug_gram_dev": (C.c_int, [_P, _P, C.c_int, _U64, _U64, _U64, C.c_int, _P, _P, C.c_int, _P,
                                      _P, _P, _P, C.c_int, C.c_int, C.c_int64]),
    "ocwg_jointq_refine": (C.c_int, [_P, _P, _U64, _U64, _P, _U64, C.POINTER(_QCfg), _P, _P, _P,
                                     C.c_double, C.c_int, C.c_int, _P, _U64, _P, _P, _P]),
    "ocwg_jointq_objective": (C.c_int, [_P, _P, _P, _P, _P, _U64, _U64, _P, _U64, C.POINTER(_QCfg),
                                        C.c_double, _P]),
    "ocwg_jointq_optimal_group_scale": (C.c_int, [_P, _P, _P, _P, _P, _U64, _U64, _P, _U64,
                                                  C.POINTER(_QCfg), C.c_double, _U64, _P]),
    "ocwg_launch_count": (_U64, [_P]),
    "ocwg_debug_profile": (C.c_int, [_P, C.c_int, _P]),
    "ocwg_debug_gemm": (C.c_int, [_P, C.c_int, _U64, _U64, _U64, C.c_double, _P, _U64, C.c_int, _P,
                                  _U64, C.c_int, C.c_double, _P, _U64, C.c_int, C.c_int, _P]),
}

_lib = None


def lib() -> C.CDLL:
    """Load libocwg.so (fails loudly when the CUDA library was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise CudaError(f"libocwg.so not built at {LIB_PATH}: run __graft_entry__.build()")
        l = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(l, name)
            fn.restype = res
            fn.argtypes = args
        _lib = l
    return _lib


def _check(status: int) -> None:
    if status != 0:
        msg = lib().ocwg_last_error().decode(errors="replace")
        raise _ERRORS.get(status, CudaError)(msg)


class Context:
    """One ocwg context (CUDA device, stream, workspace) -- ocwg_create."""

    def __init__(self, device: int = 0):
        h = _P()
        _check(lib().ocwg_create(int(device), C.byref(h)))
        self.handle = h
        self.device = device

    def close(self) -> None:
        if self.handle:
            lib().ocwg_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter teardown
        try:
            self.close()
        except Exception:
            pass


_contexts: dict[int, Context] = {}


def context(device: int = 0) -> Context:
    if device not in _contexts:
        _contexts[device] = Context(device)
    return _contexts[device]


FP32, FP64 = 0, 1


def set_precision(precision: int, device: int = 0) -> None:
    """Arithmetic of the factorisation + GPTQ sweep: FP32 (default, fast) or
    FP64 (the reference's arithmetic class, layerwise.cpp:31-90)."""
    _check(lib().ocwg_set_precision(context(device).handle, int(precision)))


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


# ------------------------------------------------------------------ quant.hpp
def quant_group_count(cfg: QuantConfig, rows: int, cols: int) -> int:
    c = cfg._c()
    return int(lib().ocwg_group_count(C.byref(c), rows, cols))


def uniform_storage_bytes(cfg: QuantConfig, rows: int, cols: int) -> int:
    c = cfg._c()
    return int(lib().ocwg_storage_bytes(C.byref(c), rows, cols))


def storage_bytes(q: QuantizedMatrix) -> int:
    return uniform_storage_bytes(q.config, q.rows, q.cols)


def validate_config(cfg: QuantConfig) -> None:
    c = cfg._c()
    _check(lib().ocwg_validate_config(C.byref(c)))


def calibrate_grids(w, cfg: QuantConfig, mode: ScaleMode = ScaleMode.minmax, device: int = 0):
    w = _f32(w)
    rows, cols = w.shape
    c = cfg._c()
    ng = quant_group_count(cfg, rows, cols)
    s = np.zeros(ng, np.float32)
    z = np.zeros(ng, np.int32)
    _check(lib().ocwg_calibrate_grids(context(device).handle, _ptr(w), rows, cols, C.byref(c),
                                      int(mode), _ptr(s), _ptr(z)))
    return s, z


def quantize_matrix(w, cfg: QuantConfig, mode: ScaleMode = ScaleMode.minmax,
                    device: int = 0) -> QuantizedMatrix:
    w = _f32(w)
    rows, cols = w.shape
    c = cfg._c()
    ng = quant_group_count(cfg, rows, cols)
    codes = np.zeros((rows, cols), np.int16)
    s = np.zeros(ng, np.float32)
    z = np.zeros(ng, np.int32)
    _check(lib().ocwg_quantize_matrix(context(device).handle, _ptr(w), rows, cols, C.byref(c),
                                      int(mode), _ptr(codes), _ptr(s), _ptr(z)))
    return QuantizedMatrix(rows, cols, cfg, codes, s, z)


def dequantize(q: QuantizedMatrix, device: int = 0) -> np.ndarray:
    c = q.config._c()
    out = np.zeros((q.rows, q.cols), np.float32)
    codes = np.ascontiguousarray(q.codes, np.int16)
    s = np.ascontiguousarray(q.scales, np.float32)
    z = np.ascontiguousarray(q.zeros, np.int32)
    _check(lib().ocwg_dequantize(context(device).handle, _ptr(codes), _ptr(s), _ptr(z), q.rows,
                                 q.cols, C.byref(c), _ptr(out)))
    return out


def activation_objective(w, w_hat, h, device: int = 0) -> float:
    w, w_hat, h = _f32(w), _f32(w_hat), _f32(h)
    if w.shape != w_hat.shape:
        raise InvalidInput("activation_objective: shape mismatch")
    if h.shape[0] != h.shape[1] or h.shape[0] != w.shape[0]:
        raise InvalidInput("activation_objective: H must be N x N with N = rows of W")
    out = C.c_double()
    _check(lib().ocwg_activation_objective(context(device).handle, _ptr(w), _ptr(w_hat), _ptr(h),
                                           w.shape[0], w.shape[1], C.byref(out)))
    return float(out.value)


# ------------------------------------------------------------------ jointq.hpp
@dataclass
class JointqOptions:
    """jointq.hpp:9-13"""
    lambda_: float = 0.2
    max_passes: int = 8
    move_radius: int = 1


@dataclass
class JointqResult:
    """jointq.hpp:27-32"""
    refined: "QuantizedMatrix"
    objective_trace: np.ndarray
    accepted_moves: int
    passes: int


def _jq_inputs(q: "QuantizedMatrix", w, x):
    w, x = _f32(w), _f32(x)
    if w.shape != (q.rows, q.cols):
        raise InvalidInput("jointq: quantized shape does not match W")
    if x.ndim != 2 or x.shape[1] != w.shape[0]:
        raise InvalidInput("jointq: X cols must equal W rows")
    codes = np.ascontiguousarray(q.codes, np.int16).reshape(q.rows, q.cols)
    return (w, x, codes.copy(), np.ascontiguousarray(q.scales, np.float32).copy(),
            np.ascontiguousarray(q.zeros, np.int32).copy())


def jointq_objective(q: "QuantizedMatrix", w, x, lambda_: float, device: int = 0) -> float:
    """jointq_objective (jointq.cpp:160-167): ||X What - X W||^2 + n lambda ||What - W||^2."""
    w, x, codes, s, z = _jq_inputs(q, w, x)
    c = q.config._c()
    out = C.c_double()
    _check(lib().ocwg_jointq_objective(context(device).handle, _ptr(codes), _ptr(s), _ptr(z), _ptr(w),
                                       q.rows, q.cols, _ptr(x), x.shape[0], C.byref(c), lambda_,
                                       C.byref(out)))
    return float(out.value)


def jointq_optimal_group_scale(q: "QuantizedMatrix", w, x, lambda_: float, group: int,
                               device: int = 0) -> float:
    """jointq_optimal_group_scale (jointq.cpp:169-175)."""
    w, x, codes, s, z = _jq_inputs(q, w, x)
    c = q.config._c()
    out = C.c_double()
    _check(lib().ocwg_jointq_optimal_group_scale(context(device).handle, _ptr(codes), _ptr(s), _ptr(z),
                                                 _ptr(w), q.rows, q.cols, _ptr(x), x.shape[0],
                                                 C.byref(c), lambda_, group, C.byref(out)))
    return float(out.value)


def jointq_refine(q0: "QuantizedMatrix", w, x, opts: JointqOptions = JointqOptions(),
                  device: int = 0) -> JointqResult:
    """jointq_refine (jointq.cpp:177-255) on the GPU (csrc/jointq.cu)."""
    w, x, codes, s, z = _jq_inputs(q0, w, x)
    c = q0.config._c()
    # at most one accepted move per group refit, cell and zero step per pass
    bound = max(0, opts.max_passes) * (q0.rows * q0.cols + 2 * len(s)) + 1
    trace = np.zeros(min(bound, 1 << 24), np.float64)
    tlen, acc, passes = C.c_uint64(), C.c_uint64(), C.c_int()
    _check(lib().ocwg_jointq_refine(context(device).handle, _ptr(w), q0.rows, q0.cols, _ptr(x),
                                    x.shape[0], C.byref(c), _ptr(codes), _ptr(s), _ptr(z),
                                    opts.lambda_, opts.max_passes, opts.move_radius, _ptr(trace),
                                    trace.size, C.byref(tlen), C.byref(acc), C.byref(passes)))
    if tlen.value == 0 or tlen.value > trace.size:
        raise CudaError(f"jointq_refine: objective trace unavailable ({tlen.value} entries)")
    refined = QuantizedMatrix(q0.rows, q0.cols, q0.config, codes, s, z)
    return JointqResult(refined, trace[:tlen.value].copy(), int(acc.value), int(passes.value))


# ------------------------------------------------------------------ OCW1 uniform payload
def pack_uniform(q: QuantizedMatrix, device: int = 0) -> bytes:
    c = q.config._c()
    n = uniform_storage_bytes(q.config, q.rows, q.cols)
    out = np.zeros(max(n, 1), np.uint8)
    codes = np.ascontiguousarray(q.codes, np.int16)
    _check(lib().ocwg_pack_uniform(context(device).handle, _ptr(codes), _ptr(_f32(q.scales)),
                                   _ptr(np.ascontiguousarray(q.zeros, np.int32)), q.rows, q.cols,
                                   C.byref(c), _ptr(out), n))
    return out[:n].tobytes()


def unpack_uniform(payload: bytes, rows: int, cols: int, cfg: QuantConfig,
                   device: int = 0) -> QuantizedMatrix:
    c = cfg._c()
    buf = np.frombuffer(payload, np.uint8).copy()
    ng = quant_group_count(cfg, rows, cols)
    codes = np.zeros((rows, cols), np.int16)
    s = np.zeros(ng, np.float32)
    z = np.zeros(ng, np.int32)
    _check(lib().ocwg_unpack_uniform(context(device).handle, _ptr(buf), len(payload), rows, cols,
                                     C.byref(c), _ptr(codes), _ptr(s), _ptr(z)))
    return QuantizedMatrix(rows, cols, cfg, codes, s, z)


# ------------------------------------------------------------------ stats.hpp
def accumulate_stats(stats: CalibStats, x_fp, x_pert, device: int = 0) -> None:
    x_fp = _f32(x_fp)
    same = x_pert is x_fp
    x_pert = x_fp if same else _f32(x_pert)
    if x_fp.shape != x_pert.shape:
        raise InvalidInput(f"accumulate_stats: shape mismatch ({x_fp.shape} vs {x_pert.shape})")
    if x_fp.shape[1] != stats.dim():
        raise InvalidInput(f"accumulate_stats: stats dimension {stats.dim()} does not match "
                           f"inputs with {x_fp.shape[1]} columns")
    gram = np.ascontiguousarray(stats.gram, np.float64)
    cross = np.ascontiguousarray(stats.cross, np.float64)
    tc = C.c_uint64(stats.token_count)
    _check(lib().ocwg_accumulate_stats(context(device).handle, _ptr(x_fp), _ptr(x_pert),
                                       x_fp.shape[0], x_fp.shape[1], _ptr(gram), _ptr(cross),
                                       C.byref(tc)))
    stats.gram, stats.cross, stats.token_count = gram, cross, int(tc.value)


def hessian_bf16(x_bf16_bits: np.ndarray, h: np.ndarray | None = None, device: int = 0) -> np.ndarray:
    """H (+)= X^T X for bf16 tokens (uint16 bit patterns, T x N) on the tensor cores."""
    x = np.ascontiguousarray(x_bf16_bits, np.uint16)
    t, n = x.shape
    acc = h is not None
    out = np.ascontiguousarray(h, np.float32).copy() if acc else np.zeros((n, n), np.float32)
    _check(lib().ocwg_hessian_bf16(context(device).handle, _ptr(x), t, n, _ptr(out), int(acc)))
    return out


# ------------------------------------------------------------------ layerwise.hpp
def gptq_order(h, actorder: bool, device: int = 0) -> np.ndarray:
    h = _f32(h)
    n = h.shape[0]
    out = np.zeros(n, np.int64)
    _check(lib().ocwg_gptq_order(context(device).handle, _ptr(h), n, int(bool(actorder)), _ptr(out)))
    return out


def _check_shapes(w: np.ndarray, h: np.ndarray) -> None:
    if h.ndim != 2 or h.shape[0] != h.shape[1] or h.shape[0] != w.shape[0]:
        raise InvalidInput("gptq_quantize: H must be N x N with N = rows of W")


def gptq_quantize(w, h, cfg: QuantConfig, opts: GptqOptions = GptqOptions(),
                  mode: ScaleMode = ScaleMode.minmax, want_w_hat: bool = False,
                  device: int = 0) -> QuantizedMatrix:
    w, h = _f32(w), _f32(h)
    validate_config(cfg)
    _check_shapes(w, h)
    n, m = w.shape
    ng = quant_group_count(cfg, n, m)
    codes = np.zeros((n, m), np.int16)
    s = np.zeros(ng, np.float32)
    z = np.zeros(ng, np.int32)
    wh = np.zeros((n, m), np.float32) if want_w_hat else None
    c, o = cfg._c(), opts._c()
    _check(lib().ocwg_gptq_quantize(context(device).handle, _ptr(w), _ptr(h), n, m, C.byref(c),
                                    C.byref(o), int(mode), _ptr(codes), _ptr(s), _ptr(z), _ptr(wh)))
    return QuantizedMatrix(n, m, cfg, codes, s, z, wh)


def gptq_factor(h, actorder: bool, percdamp: float, device: int = 0):
    """(order, hinv, U, damp) of layerwise.cpp:29-51, computed on the GPU."""
    h = _f32(h)
    n = h.shape[0]
    order = np.zeros(n, np.int64)
    hinv = np.zeros((n, n), np.float64)
    u = np.zeros((n, n), np.float64)
    damp = C.c_double()
    _check(lib().ocwg_gptq_factor(context(device).handle, _ptr(h), n, int(bool(actorder)),
                                  float(percdamp), _ptr(order), _ptr(hinv), _ptr(u), C.byref(damp)))
    return order, hinv, u, float(damp.value)


def qep_target(w, stats: CalibStats, opts: QepOptions, device: int = 0) -> np.ndarray:
    """layerwise.cpp:95-112: W + alpha (gram + lambda I)^-1 (cross W), fp64 on the GPU."""
    w = _f32(w)
    if stats.dim() != w.shape[0]:
        raise InvalidInput("qep_target: stats dimension does not match W rows")
    gram = np.ascontiguousarray(stats.gram, np.float64)
    cross = np.ascontiguousarray(stats.cross, np.float64)
    out = np.empty_like(w)
    _check(lib().ocwg_qep_target(context(device).handle, _ptr(w), _ptr(gram), _ptr(cross),
                                 w.shape[0], w.shape[1], float(opts.alpha), float(opts.eta),
                                 _ptr(out)))
    return out


def base_method_from_name(name: str) -> str:
    """layerwise.cpp:114-118."""
    if name in ("rtn", "gptq"):
        return name
    raise InvalidInput(f"unknown quantization method: {name}")


class _QepOpt(C.Structure):
    _fields_ = [("alpha", C.c_double), ("eta", C.c_double)]


def quantize_layer(w, stats: CalibStats, opts: LayerQuantOptions, device: int = 0,
                   want_w_hat: bool = False) -> QuantizedMatrix:
    """layerwise.cpp:120-126: [qep_target] -> RTN or GPTQ on stats.gram_matrix(),
    in one device round trip (ocwg_quantize_layer)."""
    w = _f32(w)
    method = base_method_from_name(opts.method)
    n, m = w.shape
    if method == "rtn" and opts.qep is None:  # quantize_matrix ignores the statistics
        q = quantize_matrix(w, opts.config, opts.scale_mode, device)
        if want_w_hat:
            q.w_hat = dequantize(q, device)
        return q
    if stats.dim() != n:
        raise InvalidInput("qep_target: stats dimension does not match W rows" if opts.qep is not None
                           else "gptq_quantize: H must be N x N with N = rows of W")
    gram = np.ascontiguousarray(stats.gram, np.float64)
    cross = np.ascontiguousarray(stats.cross, np.float64) if opts.qep is not None else None
    qep = _QepOpt(float(opts.qep.alpha), float(opts.qep.eta)) if opts.qep is not None else None
    cfg = opts.config
    ng = quant_group_count(cfg, n, m)
    codes = np.zeros((n, m), np.int16)
    scales = np.zeros(ng, np.float32)
    zeros = np.zeros(ng, np.int32)
    w_hat = np.zeros((n, m), np.float32) if want_w_hat else None
    c, o = cfg._c(), opts.gptq._c()
    _check(lib().ocwg_quantize_layer(context(device).handle, _ptr(w), _ptr(gram), _ptr(cross), n, m,
                                     1 if method == "gptq" else 0, C.byref(c), C.byref(o),
                                     int(opts.scale_mode), C.byref(qep) if qep is not None else None,
                                     _ptr(codes), _ptr(scales), _ptr(zeros), _ptr(w_hat)))
    return QuantizedMatrix(n, m, cfg, codes, scales, zeros, w_hat)


class LayerOutputs:
    """Caller-owned host buffers for quantize_layer_x (e.g. views of pinned
    memory, so the device-to-host copies run at full PCIe rate)."""

    def __init__(self, n: int, m: int, cfg: QuantConfig, alloc=np.zeros, with_h: bool = True,
                 with_w_hat: bool = True):
        ng = quant_group_count(cfg, n, m)
        self.payload_bytes = uniform_storage_bytes(cfg, n, m)
        self.codes = alloc((n, m), np.int16)
        self.scales = alloc(ng, np.float32)
        self.zeros = alloc(ng, np.int32)
        # (the reference's quantize_layer returns codes + grids; W_hat is the
        # separate dequantize(), so it is optional here)
        self.w_hat = alloc((n, m), np.float32) if with_w_hat else None
        self.payload = alloc(max(self.payload_bytes, 1), np.uint8)
        self.h = alloc((n, n), np.float32) if with_h else None


def candidate_grid(w, mode: str = "naive", in_diag=None, device: int = 0):
    """autobit.cpp:45-61: the default AutoBit candidate grid -- for bits 2..8 x
    {per_group 128, per_channel}, symmetric, the RTN error (estimate_error
    :16-34; mode "naive" or "act"/"act_aware") and storage cost.  Returns a
    list of (QuantConfig, cost_bytes, err) in the reference's order."""
    w = _f32(w)
    modes = {"naive": 0, "act": 1, "act_aware": 1}
    if mode not in modes:
        raise InvalidInput(f"unknown error mode: {mode}")
    if in_diag is not None:
        in_diag = np.ascontiguousarray(in_diag, np.float64)
        if in_diag.shape != (w.shape[0],):
            raise InvalidInput("estimate_error: input diagonal length mismatch")
    errs = np.zeros(14, np.float64)
    costs = np.zeros(14, np.uint64)
    _check(lib().ocwg_candidate_grid(context(device).handle, _ptr(w), w.shape[0], w.shape[1],
                                     modes[mode], _ptr(in_diag), _ptr(errs), _ptr(costs)))
    out = []
    for k in range(14):
        cfg = QuantConfig(2 + k // 2, Scheme.symmetric,
                          Granularity.per_channel if k & 1 else Granularity.per_group, 128)
        out.append((cfg, int(costs[k]), float(errs[k])))
    return out


def quantize_layers_x(ws, x_bf16_bits, cfg: QuantConfig, opts: GptqOptions,
                      mode: ScaleMode = ScaleMode.minmax, device: int = 0):
    """Layers that share one calibration input (q/k/v, gate/up):
    one Hessian and one factorisation, then a sweep per W.  Returns one
    (QuantizedMatrix, payload bytes) per W, equal to separate quantize_layer_x
    calls."""
    ws = [_f32(w) for w in ws]
    x = np.ascontiguousarray(x_bf16_bits, np.uint16)
    if not ws:
        raise InvalidInput("quantize_layers_x: no layers")
    n = ws[0].shape[0]
    if any(w.shape[0] != n for w in ws) or x.shape[1] != n:
        raise InvalidInput("quantize_layers_x: every W must be N x M_i with N = columns of X")
    k = len(ws)
    outs = []
    for w in ws:
        m = w.shape[1]
        ng = quant_group_count(cfg, n, m)
        outs.append((np.zeros((n, m), np.int16), np.zeros(ng, np.float32), np.zeros(ng, np.int32),
                     np.zeros(max(uniform_storage_bytes(cfg, n, m), 1), np.uint8)))
    arr = lambda vals, t: (t * k)(*vals)  # noqa: E731
    wp = arr([w.ctypes.data for w in ws], C.c_void_p)
    mp = arr([w.shape[1] for w in ws], C.c_uint64)
    cp = arr([o[0].ctypes.data for o in outs], C.c_void_p)
    sp = arr([o[1].ctypes.data for o in outs], C.c_void_p)
    zp = arr([o[2].ctypes.data for o in outs], C.c_void_p)
    pp = arr([o[3].ctypes.data for o in outs], C.c_void_p)
    pl = arr([o[3].size for o in outs], C.c_uint64)
    c, o = cfg._c(), opts._c()
    _check(lib().ocwg_quantize_layers_x(context(device).handle, k, C.cast(wp, C.c_void_p),
                                        C.cast(mp, C.c_void_p), _ptr(x), x.shape[0], n,
                                        C.byref(c), C.byref(o), int(mode), C.cast(cp, C.c_void_p),
                                        C.cast(sp, C.c_void_p), C.cast(zp, C.c_void_p),
                                        C.cast(pp, C.c_void_p), C.cast(pl, C.c_void_p)))
    res = []
    for w, (codes, s_, z_, pay) in zip(ws, outs):
        pb = uniform_storage_bytes(cfg, n, w.shape[1])
        res.append((QuantizedMatrix(n, w.shape[1], cfg, codes, s_, z_), pay[:pb].tobytes()))
    return res


def quantize_layer_x(w, x_bf16_bits, cfg: QuantConfig, opts: GptqOptions,
                     mode: ScaleMode = ScaleMode.minmax, device: int = 0,
                     out: LayerOutputs | None = None):
    """The north_star's one-call layer quantize from host buffers:
    W (N x M fp32) + calibration tokens X (T x N bf16 bits) ->
    (QuantizedMatrix with w_hat, packed OCW1 payload bytes, H fp32 or None).
    X streams to the device in token chunks while the Hessian accumulates."""
    w = _f32(w)
    x = np.ascontiguousarray(x_bf16_bits, np.uint16)
    n, m = w.shape
    if x.shape[1] != n:
        raise InvalidInput("quantize_layer_x: X must be T x N with N = rows of W")
    o_ = out if out is not None else LayerOutputs(n, m, cfg)
    pb = o_.payload_bytes
    codes, s, z, wh, payload, h = o_.codes, o_.scales, o_.zeros, o_.w_hat, o_.payload, o_.h
    c, o = cfg._c(), opts._c()
    _check(lib().ocwg_quantize_layer_x(context(device).handle, _ptr(w), _ptr(x), x.shape[0], n, m,
                                       C.byref(c), C.byref(o), int(mode), _ptr(codes), _ptr(s),
                                       _ptr(z), _ptr(wh), _ptr(payload), pb, _ptr(h)))
    if out is not None:
        return QuantizedMatrix(n, m, cfg, codes, s, z, wh), payload[:pb], h
    return QuantizedMatrix(n, m, cfg, codes, s, z, wh), payload[:pb].tobytes(), h
