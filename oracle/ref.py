"""ctypes wrapper over oracle/_ref/libocw_ref.so -- the reference's own hot-path
sources (proj/src/{quant,stats,layerwise,matrix}.cpp) compiled unmodified by
oracle/build_ref.sh, plus oracle/ref_capi.cpp.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline / --impl reference arm.  The product package never
imports it.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_ref" / "libocw_ref.so"
_P, _U64, _I = C.c_void_p, C.c_uint64, C.c_int

_SIGS = {
    "ocwref_last_error": (C.c_char_p, []),
    "ocwref_blas_name": (C.c_char_p, []),
    "ocwref_set_threads": (None, [_I]),
    "ocwref_use_blas": (None, [_I]),
    "ocwref_group_count": (_U64, [_I, _I, _I, _U64, _U64, _U64]),
    "ocwref_storage_bytes": (_U64, [_I, _I, _I, _U64, _U64, _U64]),
    "ocwref_random_gaussian": (_I, [_U64, _U64, _U64, C.c_float, _P]),
    "ocwref_calibrate_grids": (_I, [_P, _U64, _U64, _I, _I, _I, _U64, _I, _P, _P]),
    "ocwref_quantize_matrix": (_I, [_P, _U64, _U64, _I, _I, _I, _U64, _I, _P, _P, _P]),
    "ocwref_candidate_grid": (_I, [_P, _U64, _U64, _I, _P, _P, _P]),
    "ocwref_dequantize": (_I, [_P, _P, _P, _U64, _U64, _I, _I, _I, _U64, _P]),
    "ocwref_activation_objective": (_I, [_P, _P, _P, _U64, _U64, _P]),
    "ocwref_gptq_order": (_I, [_P, _U64, _I, _P]),
    "ocwref_gptq_quantize": (_I, [_P, _P, _U64, _U64, _I, _I, _I, _U64, _I, C.c_double, _U64, _I,
                                  _P, _P, _P, _P]),
    "ocwref_gptq_factor": (_I, [_P, _U64, _I, C.c_double, _P, _P, _P]),
    "ocwref_accumulate_stats": (_I, [_P, _P, _U64, _U64, _P, _P, _P, _P]),
    "ocwref_qep_target": (_I, [_P, _P, _P, _U64, _U64, C.c_double, C.c_double, _P]),
    "ocwref_quantize_layer": (_I, [_P, _P, _P, _U64, _U64, _I, _I, _I, _I, _U64, _I, _I, C.c_double,
                                   _U64, _I, C.c_double, C.c_double, _P, _P, _P]),
    "ocwref_jointq_refine": (_I, [_P, _U64, _U64, _P, _U64, _I, _I, _I, _U64, _P, _P, _P,
                                  C.c_double, _I, _I, _P, _U64, _P, _P, _P]),
    "ocwref_jointq_objective": (_I, [_P, _P, _P, _P, _U64, _U64, _P, _U64, _I, _I, _I, _U64,
                                     C.c_double, _P]),
    "ocwref_jointq_optimal_group_scale": (_I, [_P, _P, _P, _P, _U64, _U64, _P, _U64, _I, _I, _I,
                                               _U64, C.c_double, _U64, _P]),
}

_lib = None


class RefError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[{status}] {msg}")
        self.status = status


def available() -> bool:
    return LIB.exists()


def build() -> None:
    subprocess.run(["bash", str(HERE / "build_ref.sh")], check=True)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        l = C.CDLL(str(LIB))
        for name, (res, args) in _SIGS.items():
            fn = getattr(l, name)
            fn.restype = res
            fn.argtypes = args
        _lib = l
    return _lib


def _ck(st: int) -> None:
    if st != 0:
        raise RefError(st, lib().ocwref_last_error().decode())


def _p(a):
    return None if a is None else a.ctypes.data


def _f32(a):
    return np.ascontiguousarray(a, np.float32)


def random_gaussian(rows: int, cols: int, seed: int, stddev: float = 1.0) -> np.ndarray:
    """matrix.cpp:57-62 (the reference's seeded fixture generator)."""
    out = np.zeros((rows, cols), np.float32)
    _ck(lib().ocwref_random_gaussian(rows, cols, seed, stddev, _p(out)))
    return out


def group_count(bits, scheme, gran, group, rows, cols) -> int:
    return int(lib().ocwref_group_count(bits, scheme, gran, group, rows, cols))


def storage_bytes(bits, scheme, gran, group, rows, cols) -> int:
    return int(lib().ocwref_storage_bytes(bits, scheme, gran, group, rows, cols))


def calibrate_grids(w, bits, scheme, gran, group, mse=False):
    w = _f32(w)
    ng = group_count(bits, scheme, gran, group, *w.shape)
    s, z = np.zeros(ng, np.float32), np.zeros(ng, np.int32)
    _ck(lib().ocwref_calibrate_grids(_p(w), w.shape[0], w.shape[1], bits, scheme, gran, group,
                                     int(mse), _p(s), _p(z)))
    return s, z


def quantize_matrix(w, bits, scheme, gran, group, mse=False):
    w = _f32(w)
    ng = group_count(bits, scheme, gran, group, *w.shape)
    codes = np.zeros(w.shape, np.int16)
    s, z = np.zeros(ng, np.float32), np.zeros(ng, np.int32)
    _ck(lib().ocwref_quantize_matrix(_p(w), w.shape[0], w.shape[1], bits, scheme, gran, group,
                                     int(mse), _p(codes), _p(s), _p(z)))
    return codes, s, z


def dequantize(codes, s, z, bits, scheme, gran, group):
    codes = np.ascontiguousarray(codes, np.int16)
    out = np.zeros(codes.shape, np.float32)
    _ck(lib().ocwref_dequantize(_p(codes), _p(_f32(s)), _p(np.ascontiguousarray(z, np.int32)),
                                codes.shape[0], codes.shape[1], bits, scheme, gran, group, _p(out)))
    return out


def activation_objective(w, w_hat, h) -> float:
    w, w_hat, h = _f32(w), _f32(w_hat), _f32(h)
    out = C.c_double()
    _ck(lib().ocwref_activation_objective(_p(w), _p(w_hat), _p(h), w.shape[0], w.shape[1],
                                          C.byref(out)))
    return out.value


def gptq_order(h, actorder: bool) -> np.ndarray:
    h = _f32(h)
    out = np.zeros(h.shape[0], np.int64)
    _ck(lib().ocwref_gptq_order(_p(h), h.shape[0], int(actorder), _p(out)))
    return out


def candidate_grid(w, mode=0, in_diag=None):
    """autobit.cpp:45-61: (errors[14], cost_bytes[14]) of the default grid."""
    w = _f32(w)
    errs, costs = np.zeros(14), np.zeros(14, np.uint64)
    d = None if in_diag is None else np.ascontiguousarray(in_diag, np.float64)
    _ck(lib().ocwref_candidate_grid(_p(w), w.shape[0], w.shape[1], int(mode),
                                    None if d is None else _p(d), _p(errs), _p(costs)))
    return errs, costs


def gptq_quantize(w, h, bits, scheme, gran, group, actorder=False, percdamp=0.01, block=32,
                  mse=False, timing=False):
    w, h = _f32(w), _f32(h)
    n, m = w.shape
    ng = group_count(bits, scheme, gran, group, n, m)
    codes = np.zeros((n, m), np.int16)
    s, z = np.zeros(ng, np.float32), np.zeros(ng, np.int32)
    sec = C.c_double()
    _ck(lib().ocwref_gptq_quantize(_p(w), _p(h), n, m, bits, scheme, gran, group, int(actorder),
                                   percdamp, block, int(mse), _p(codes), _p(s), _p(z),
                                   C.byref(sec)))
    return (codes, s, z, sec.value) if timing else (codes, s, z)


def gptq_factor(h, actorder=False, percdamp=0.01):
    h = _f32(h)
    n = h.shape[0]
    hinv, u = np.zeros((n, n)), np.zeros((n, n))
    damp = C.c_double()
    _ck(lib().ocwref_gptq_factor(_p(h), n, int(actorder), percdamp, _p(hinv), _p(u), C.byref(damp)))
    return hinv, u, damp.value


def accumulate_stats(gram, cross, x_fp, x_pert, token_count=0, timing=False):
    """In-place on fp64 gram/cross (row-major)."""
    x_fp, x_pert = _f32(x_fp), _f32(x_pert)
    tc = C.c_uint64(token_count)
    sec = C.c_double()
    _ck(lib().ocwref_accumulate_stats(_p(x_fp), _p(x_pert), x_fp.shape[0], x_fp.shape[1], _p(gram),
                                      _p(cross), C.byref(tc), C.byref(sec)))
    return (int(tc.value), sec.value) if timing else int(tc.value)


def qep_target(w, gram, cross, alpha=1.0, eta=0.01):
    """layerwise.cpp:95-112 (the reference's own qep_target)."""
    w = _f32(w)
    out = np.empty_like(w)
    _ck(lib().ocwref_qep_target(_p(w), _p(np.ascontiguousarray(gram, np.float64)),
                                _p(np.ascontiguousarray(cross, np.float64)), w.shape[0], w.shape[1],
                                float(alpha), float(eta), _p(out)))
    return out


def quantize_layer(w, gram, cross, method_gptq, bits, scheme, gran, group, mse=False,
                   actorder=False, percdamp=0.01, block=32, qep=None):
    w = _f32(w)
    n, m = w.shape
    ng = group_count(bits, scheme, gran, group, n, m)
    codes = np.zeros((n, m), np.int16)
    s, z = np.zeros(ng, np.float32), np.zeros(ng, np.int32)
    alpha, eta = qep if qep is not None else (1.0, 0.01)
    _ck(lib().ocwref_quantize_layer(_p(w), _p(np.ascontiguousarray(gram, np.float64)),
                                    _p(None if cross is None else np.ascontiguousarray(cross, np.float64)),
                                    n, m, int(method_gptq), bits, scheme, gran, group, int(mse),
                                    int(actorder), percdamp, block, int(qep is not None), alpha, eta,
                                    _p(codes), _p(s), _p(z)))
    return codes, s, z


def use_blas(on: bool) -> None:
    """BLAS-backed shim GEMM/LLT (fast) vs fixed-order loops (bit-portable)."""
    lib().ocwref_use_blas(int(bool(on)))


def set_threads(n: int) -> None:
    lib().ocwref_set_threads(int(n))


def blas_name() -> str:
    return lib().ocwref_blas_name().decode()


# ---- the reference's own OCW1 container (src/container.cpp), SURVEY §8 f2 ----
CONTAINER_LIB = HERE / "_ref" / "libocw_ref_container.so"
_clib = None


def container_lib():
    """libocw_ref_container.so, or None when the image lacks nlohmann/json."""
    global _clib
    if _clib is None and CONTAINER_LIB.exists():
        l = C.CDLL(str(CONTAINER_LIB))
        l.ocwref_container_error.restype = C.c_char_p
        l.ocwref_serialize_ocw.restype = _I
        l.ocwref_roundtrip_ocw.restype = _I
        _clib = l
    return _clib


def _arr(vals, t):
    return (t * len(vals))(*vals)


def serialize_ocw(records, meta_json: str | None = None) -> bytes:
    """serialize_ocw (container.cpp:344-373) over records of
    ("f32", name, array) or ("uniform", name, codes, scales, zeros, bits, scheme, gran, group)."""
    l = container_lib()
    k = len(records)
    keep = []
    names, kind, rows, cols, bits, sch, gran, grp, f32, cds, scs, zrs = ([] for _ in range(12))
    for r in records:
        names.append(r[1].encode())
        if r[0] == "f32":
            a = np.ascontiguousarray(r[2], np.float32)
            keep.append(a)
            kind.append(0), rows.append(a.shape[0]), cols.append(a.shape[1])
            bits.append(0), sch.append(0), gran.append(0), grp.append(0)
            f32.append(a.ctypes.data), cds.append(None), scs.append(None), zrs.append(None)
        else:
            c = np.ascontiguousarray(r[2], np.int16)
            s = np.ascontiguousarray(r[3], np.float32)
            z = np.ascontiguousarray(r[4], np.int32)
            keep += [c, s, z]
            kind.append(1), rows.append(c.shape[0]), cols.append(c.shape[1])
            bits.append(r[5]), sch.append(r[6]), gran.append(r[7]), grp.append(r[8])
            f32.append(None), cds.append(c.ctypes.data), scs.append(s.ctypes.data)
            zrs.append(z.ctypes.data)
    cap = 64 + 1024 * (k + 1) + sum(a.nbytes for a in keep) * 2 + (len(meta_json or "") * 2)
    out = np.zeros(cap, np.uint8)
    ln = C.c_size_t()
    st = l.ocwref_serialize_ocw(
        k, _arr(names, C.c_char_p), _arr(kind, C.c_int), _arr(rows, C.c_size_t),
        _arr(cols, C.c_size_t), _arr(bits, C.c_int), _arr(sch, C.c_int), _arr(gran, C.c_int),
        _arr(grp, C.c_size_t), _arr(f32, C.c_void_p), _arr(cds, C.c_void_p),
        _arr(scs, C.c_void_p), _arr(zrs, C.c_void_p),
        None if meta_json is None else meta_json.encode(), out.ctypes.data_as(C.c_void_p),
        C.c_size_t(cap), C.byref(ln))
    if st != 0:
        raise RuntimeError(l.ocwref_container_error().decode())
    return out[:ln.value].tobytes()


def roundtrip_ocw(data: bytes) -> bytes:
    """serialize_ocw(deserialize_ocw(data)) -- the reference's parser."""
    l = container_lib()
    src = np.frombuffer(data, np.uint8).copy()
    cap = len(data) * 2 + 4096
    out = np.zeros(cap, np.uint8)
    ln = C.c_size_t()
    st = l.ocwref_roundtrip_ocw(src.ctypes.data_as(C.c_void_p), C.c_size_t(len(data)),
                                out.ctypes.data_as(C.c_void_p), C.c_size_t(cap), C.byref(ln))
    if st != 0:
        raise RuntimeError(l.ocwref_container_error().decode())
    return out[:ln.value].tobytes()


# ---------------------------------------------------------------- jointq.cpp
def jointq_refine(codes, scales, zeros, w, x, bits, scheme, gran, group, lambda_=0.2,
                  max_passes=8, radius=1, trace_cap=1 << 20):
    """jointq.cpp:177-255: (codes, scales, zeros, trace, accepted_moves, passes)."""
    w, x = _f32(w), _f32(x)
    codes = np.ascontiguousarray(codes, np.int16).copy()
    s, z = _f32(scales).copy(), np.ascontiguousarray(zeros, np.int32).copy()
    trace = np.zeros(trace_cap, np.float64)
    tl, acc, ps = C.c_size_t(), C.c_size_t(), C.c_int()
    _ck(lib().ocwref_jointq_refine(_p(w), w.shape[0], w.shape[1], _p(x), x.shape[0], bits, scheme,
                                   gran, group, _p(codes), _p(s), _p(z), lambda_, max_passes, radius,
                                   _p(trace), trace_cap, C.byref(tl), C.byref(acc), C.byref(ps)))
    return codes, s, z, trace[:min(tl.value, trace_cap)].copy(), int(acc.value), int(ps.value)


def jointq_objective(codes, scales, zeros, w, x, bits, scheme, gran, group, lambda_) -> float:
    w, x = _f32(w), _f32(x)
    out = C.c_double()
    _ck(lib().ocwref_jointq_objective(_p(np.ascontiguousarray(codes, np.int16)), _p(_f32(scales)),
                                      _p(np.ascontiguousarray(zeros, np.int32)), _p(w), w.shape[0],
                                      w.shape[1], _p(x), x.shape[0], bits, scheme, gran, group,
                                      lambda_, C.byref(out)))
    return float(out.value)


def jointq_optimal_group_scale(codes, scales, zeros, w, x, bits, scheme, gran, group, lambda_,
                               g) -> float:
    w, x = _f32(w), _f32(x)
    out = C.c_double()
    _ck(lib().ocwref_jointq_optimal_group_scale(
        _p(np.ascontiguousarray(codes, np.int16)), _p(_f32(scales)),
        _p(np.ascontiguousarray(zeros, np.int32)), _p(w), w.shape[0], w.shape[1], _p(x), x.shape[0],
        bits, scheme, gran, group, lambda_, g, C.byref(out)))
    return float(out.value)
