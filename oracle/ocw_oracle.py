"""CPU oracle for the OneComp (ocw) GPTQ layer-quantize hot path.

TEST INFRASTRUCTURE ONLY. This module is the *checker*: it restates, in numpy
(fp64 where the reference uses Eigen ``MatrixXd``, fp32 where it uses
``float``), the reference algorithm of the path this repository accelerates.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` arm may import it.  The product path
(``paper_2603_28845_b200``) never imports or calls it.

Parity pin: the restatement is checked against
  * every known-answer / exact-equivalence test the reference holds for this
    path (proj/tests/test_core.cpp, proj/tests/test_layerwise.cpp,
    proj/tests/test_pipeline.cpp:93-114), ported in tests/test_oracle_*.py, and
  * golden vectors produced by the reference's *own* sources compiled here
    (oracle/build_ref.sh -> oracle/_ref, fixtures in tests/golden/).

All citations are relative to /root/reference/proj/.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np

# --------------------------------------------------------------------------
# errors (include/ocw/errors.hpp:9-21)
# --------------------------------------------------------------------------


class InvalidInput(ValueError):
    """ocw::invalid_input (errors.hpp:9-11)."""


class NumericError(RuntimeError):
    """ocw::numeric_error (errors.hpp:19-21)."""


# --------------------------------------------------------------------------
# fp16 (include/ocw/fp16.hpp:12-75) -- the reference's own integer routine.
# It is IEEE-exact for normal halves but NOT in the subnormal-half range
# (|x| < 2^-14): the encoder's subnormal branch keeps one bit too few and the
# decoder then re-normalises with an off-by-one exponent.  We restate it bit
# for bit, quirk included.
# --------------------------------------------------------------------------

K_FP16_MIN_POSITIVE = np.float32(5.9604644775390625e-08)  # fp16.hpp:75


def fp16_encode(f) -> np.ndarray:
    """fp16.hpp:12-45, vectorised."""
    f = np.asarray(f, dtype=np.float32)
    x = f.view(np.uint32).astype(np.uint64)
    sign = (x >> 16) & 0x8000
    x = x & 0x7FFFFFFF
    out = np.zeros(x.shape, dtype=np.uint64)

    big = x >= 0x47800000                               # :16-19
    out = np.where(big & (x > 0x7F800000), sign | 0x7E00, out)
    out = np.where(big & (x <= 0x7F800000), sign | 0x7C00, out)

    sub = (~big) & (x < 0x38800000)                      # :20-30
    tiny = sub & (x < 0x33000000)
    out = np.where(tiny, sign, out)
    ss = sub & ~tiny
    shift = np.where(ss, 126 - (x >> 23).astype(np.int64), 1).astype(np.uint64)
    mant = (x & 0x7FFFFF) | 0x800000
    rounded = mant >> (shift + 1)
    round_bit = (mant >> shift) & 1
    sticky = (mant & ((np.uint64(1) << shift) - 1)) != 0
    rounded = rounded + ((round_bit == 1) & (sticky | ((rounded & 1) == 1))).astype(np.uint64)
    out = np.where(ss, sign | rounded, out)

    nrm = (~big) & ~sub                                 # :32-44
    m = x & 0x7FFFFF
    e = ((x >> 23).astype(np.int64) - 127 + 15)
    e = np.where(nrm, e, 0).astype(np.uint64)
    h = (sign | (e << 10) | (m >> 13)) & 0xFFFF
    rb = (m >> 12) & 1
    st = (m & 0xFFF) != 0
    h = h + ((rb == 1) & (st | ((h & 1) == 1))).astype(np.uint64)
    h = np.where((h & 0x7FFF) >= 0x7C00, sign | 0x7C00, h)
    out = np.where(nrm, h, out)
    return out.astype(np.uint16)


def fp16_decode(h) -> np.ndarray:
    """fp16.hpp:47-72, vectorised (including its subnormal normalisation)."""
    h = np.asarray(h, dtype=np.uint16).astype(np.uint64)
    sign = (h & 0x8000) << 16
    exp = (h >> 10) & 0x1F
    mant = h & 0x3FF
    out = np.zeros(h.shape, dtype=np.uint64)
    # exp == 0, mant == 0: signed zero
    out = np.where((exp == 0) & (mant == 0), sign, out)
    # exp == 0, mant != 0: loop  e=-1; while !(m & 0x400) { m <<= 1; e--; }
    sub = (exp == 0) & (mant != 0)
    msafe = np.where(sub, mant, 1).astype(np.uint64)
    # number of left shifts needed so that bit 10 is set
    nshift = np.zeros(h.shape, dtype=np.int64)
    mm = msafe.copy()
    for _ in range(11):
        need = (mm & 0x400) == 0
        mm = np.where(need, mm << 1, mm)
        nshift = nshift + need.astype(np.int64)
    e = -1 - nshift
    xsub = sign | (((127 - 15 + e + 1).astype(np.uint64) & 0xFF) << 23) | ((mm & 0x3FF) << 13)
    out = np.where(sub, xsub, out)
    inf = exp == 31
    out = np.where(inf, sign | 0x7F800000 | (mant << 13), out)
    nrm = (exp != 0) & (exp != 31)
    out = np.where(nrm, sign | (((exp + 127 - 15) & 0xFF) << 23) | (mant << 13), out)
    return out.astype(np.uint32).view(np.float32)


def fp16_round(f) -> np.ndarray:
    """fp16.hpp:71-72."""
    return fp16_decode(fp16_encode(f))


def positive_fp16(s) -> np.ndarray:
    """quant.cpp:39-42: fp16-round, floor at 2^-24 when it collapses to <= 0."""
    r = fp16_round(s)
    return np.where(r > 0, r, K_FP16_MIN_POSITIVE).astype(np.float32)


# --------------------------------------------------------------------------
# quantisation config (include/ocw/quant.hpp:12-63, quant.cpp:11-25)
# --------------------------------------------------------------------------


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


def scheme_qmin(bits: int, scheme: Scheme) -> int:
    """quant.cpp:11-13."""
    return 0 if scheme == Scheme.asymmetric else -((1 << (bits - 1)) - 1)


def scheme_qmax(bits: int, scheme: Scheme) -> int:
    """quant.cpp:15-17."""
    return (1 << bits) - 1 if scheme == Scheme.asymmetric else (1 << (bits - 1)) - 1


@dataclass
class QuantConfig:
    bits: int = 4
    scheme: Scheme = Scheme.symmetric
    granularity: Granularity = Granularity.per_group
    group_size: int = 128

    def validate(self) -> None:
        """quant.cpp:19-25."""
        if self.bits < 1 or self.bits > 8:
            raise InvalidInput("QuantConfig: bits must be in [1,8]")
        if self.scheme == Scheme.symmetric and self.bits < 2:
            raise InvalidInput("QuantConfig: symmetric grids need bits >= 2")
        if self.granularity == Granularity.per_group and self.group_size < 1:
            raise InvalidInput("QuantConfig: group_size must be >= 1")


@dataclass
class Grids:
    """std::vector<QuantGrid> in structure-of-arrays form (quant.hpp:25-30)."""
    scale: np.ndarray       # float32 [G]
    zero: np.ndarray        # int32 [G]
    qmin: int
    qmax: int

    def __len__(self) -> int:
        return len(self.scale)


@dataclass
class QuantizedMatrix:
    """quant.hpp:54-63: codes row-major int16, grids in group-index order."""
    rows: int
    cols: int
    config: QuantConfig
    codes: np.ndarray
    grids: Grids
    extra: dict = field(default_factory=dict)


def quant_groups_per_row(cfg: QuantConfig, cols: int) -> int:
    """quant.cpp:142-149."""
    if cfg.granularity == Granularity.per_tensor:
        return 0
    if cfg.granularity == Granularity.per_channel:
        return 1
    return (cols + cfg.group_size - 1) // cfg.group_size


def quant_group_count(cfg: QuantConfig, rows: int, cols: int) -> int:
    """quant.cpp:151-154."""
    if cfg.granularity == Granularity.per_tensor:
        return 1
    return rows * quant_groups_per_row(cfg, cols)


def group_index_matrix(cfg: QuantConfig, rows: int, cols: int) -> np.ndarray:
    """QuantizedMatrix::group_index (quant.cpp:158-166) for every (i, j)."""
    if cfg.granularity == Granularity.per_tensor:
        return np.zeros((rows, cols), dtype=np.int64)
    if cfg.granularity == Granularity.per_channel:
        return np.repeat(np.arange(rows, dtype=np.int64)[:, None], cols, axis=1)
    gpr = quant_groups_per_row(cfg, cols)
    return (np.arange(rows, dtype=np.int64)[:, None] * gpr
            + (np.arange(cols, dtype=np.int64)[None, :] // cfg.group_size))


# --------------------------------------------------------------------------
# scalar quantisation (quant.cpp:27-35)
# --------------------------------------------------------------------------


def _ref_int(x) -> np.ndarray:
    """int(std::nearbyint(x)) as built for x86-64: ties-to-even, and the
    float->int conversion (cvttss2si) yields INT_MIN for NaN / |x| >= 2^31."""
    with np.errstate(invalid="ignore"):
        r = np.rint(np.asarray(x, dtype=np.float32))
        ok = (r >= np.float32(-2.0**31)) & (r < np.float32(2.0**31))
    return np.where(ok, np.where(ok, r, 0), -(2**31)).astype(np.int64)


def quantize_scalar(w, scale, zero, qmin, qmax):
    """code = clamp(int(nearbyint(w / s)) + z, qmin, qmax); w_hat = s * float(code - z).

    fp32 division, ties-to-even rounding (np.rint), fp32 product.
    """
    w = np.asarray(w, dtype=np.float32)
    scale = np.asarray(scale, dtype=np.float32)
    with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
        r = _ref_int((w / scale).astype(np.float32))
    code = np.clip(r + np.asarray(zero, dtype=np.int64), qmin, qmax)
    w_hat = (scale * (code - np.asarray(zero, dtype=np.int64)).astype(np.float32)).astype(np.float32)
    return code, w_hat


def dequantize_scalar(code, scale, zero):
    """quant.cpp:33-35."""
    return (np.asarray(scale, dtype=np.float32)
            * (np.asarray(code, dtype=np.int64) - np.asarray(zero, dtype=np.int64)).astype(np.float32)
            ).astype(np.float32)


# --------------------------------------------------------------------------
# grid calibration (quant.cpp:44-196), vectorised over groups
# --------------------------------------------------------------------------


def _from_extremes(lo: np.ndarray, hi: np.ndarray, bits: int, scheme: Scheme):
    """asymmetric_from_extremes (quant.cpp:51-64) / symmetric_from_extremes (66-74)."""
    qmin, qmax = scheme_qmin(bits, scheme), scheme_qmax(bits, scheme)
    lo = lo.astype(np.float32)
    hi = hi.astype(np.float32)
    if scheme == Scheme.asymmetric:
        degen = hi == lo
        with np.errstate(all="ignore"):
            s = positive_fp16((hi - lo) / np.float32(qmax - qmin))
            s = np.where(degen, np.float32(1.0), s).astype(np.float32)
            zf = np.where(degen, np.float32(qmin) - lo, np.float32(qmin) - lo / s).astype(np.float32)
        z = np.clip(_ref_int(zf), qmin, qmax)
        return s, z.astype(np.int32)
    amax = np.maximum(np.abs(lo), np.abs(hi)).astype(np.float32)
    s = np.where(amax == 0, np.float32(1.0), positive_fp16(amax / np.float32(qmax))).astype(np.float32)
    return s, np.zeros(lo.shape, dtype=np.int32)


def _mse_refine(vals: np.ndarray, valid: np.ndarray, lo, hi, s0, z0, bits, scheme):
    """calibrate_grid_mse (quant.cpp:114-140) for a batch of groups.

    vals: [G, L] float32 padded; valid: [G, L] bool mask of real entries.
    """
    qmin, qmax = scheme_qmin(bits, scheme), scheme_qmax(bits, scheme)
    if scheme == Scheme.asymmetric:
        degen = hi == lo
        raw = (hi - lo) / np.float32(qmax - qmin)
    else:
        amax = np.maximum(np.abs(lo), np.abs(hi)).astype(np.float32)
        degen = amax == 0
        raw = amax / np.float32(qmax)
    raw = raw.astype(np.float32)

    def sq_err(s, z):
        _, wh = quantize_scalar(vals, s[:, None], z[:, None], qmin, qmax)
        d = (vals - wh).astype(np.float32).astype(np.float64)  # double(v - w_hat)
        return np.where(valid, d * d, 0.0).sum(axis=1)        # in-order sum differs only in last ulp

    best_s, best_z = s0.copy(), z0.copy()
    best_e = _ordered_sum_sq(vals, valid, s0, z0, qmin, qmax)
    for c in range(100):
        mult = np.float32(np.float32(0.3) + (np.float32(0.7) * np.float32(c)) / np.float32(99.0))
        s = positive_fp16((mult * raw).astype(np.float32))
        if scheme == Scheme.asymmetric:
            with np.errstate(all="ignore"):
                zf = (np.float32(qmin) - lo / s).astype(np.float32)
            z = np.clip(_ref_int(zf), qmin, qmax).astype(np.int32)
        else:
            z = np.zeros_like(z0)
        e = _ordered_sum_sq(vals, valid, s, z, qmin, qmax)
        better = (e < best_e) & ~degen
        best_e = np.where(better, e, best_e)
        best_s = np.where(better, s, best_s)
        best_z = np.where(better, z, best_z)
    return best_s.astype(np.float32), best_z.astype(np.int32)


def _ordered_sum_sq(vals, valid, s, z, qmin, qmax):
    """grid_sq_error (quant.cpp:85-92): sequential fp64 sum in element order."""
    _, wh = quantize_scalar(vals, s[:, None], z[:, None], qmin, qmax)
    d = (vals - wh).astype(np.float32).astype(np.float64)
    d = np.where(valid, d * d, 0.0)
    acc = np.zeros(vals.shape[0], dtype=np.float64)
    for k in range(vals.shape[1]):   # left-to-right, like the C++ loop
        acc = acc + d[:, k]
    return acc


def calibrate_grids(w: np.ndarray, cfg: QuantConfig, mode: ScaleMode = ScaleMode.minmax) -> Grids:
    """calibrate_grids (quant.cpp:168-196): grids from the ORIGINAL W, group-index order."""
    cfg.validate()
    w = np.asarray(w, dtype=np.float32)
    if w.ndim != 2:
        raise InvalidInput("calibrate_grids: expected a matrix")
    if not np.all(np.isfinite(w)):
        raise InvalidInput("calibrate_grids: non-finite entry")
    rows, cols = w.shape
    if rows == 0 or cols == 0:
        raise InvalidInput("calibrate_grids: empty matrix")
    if cfg.granularity == Granularity.per_tensor:
        vals = w.reshape(1, -1)
        valid = np.ones_like(vals, dtype=bool)
    elif cfg.granularity == Granularity.per_channel:
        vals = w
        valid = np.ones_like(vals, dtype=bool)
    else:
        G = cfg.group_size
        gpr = quant_groups_per_row(cfg, cols)
        pad = gpr * G - cols
        wp = np.pad(w, ((0, 0), (0, pad)), constant_values=np.nan)
        vals = wp.reshape(rows * gpr, G)
        valid = ~np.isnan(vals)
        vals = np.where(valid, vals, np.float32(0.0)).astype(np.float32)
    big = np.float32(np.inf)
    lo = np.where(valid, vals, big).min(axis=1)
    hi = np.where(valid, vals, -big).max(axis=1)
    s, z = _from_extremes(lo, hi, cfg.bits, cfg.scheme)
    if mode == ScaleMode.mse_grid:
        s, z = _mse_refine(vals, valid, lo, hi, s, z, cfg.bits, cfg.scheme)
    return Grids(s.astype(np.float32), z.astype(np.int32),
                 scheme_qmin(cfg.bits, cfg.scheme), scheme_qmax(cfg.bits, cfg.scheme))


def calibrate_grid(values, bits: int, scheme: Scheme, mode: ScaleMode = ScaleMode.minmax) -> Grids:
    """calibrate_asymmetric / calibrate_symmetric / calibrate_grid(_mse) (quant.cpp:96-140)."""
    values = np.asarray(values, dtype=np.float32).ravel()
    if values.size == 0:
        raise InvalidInput("calibrate: empty input")
    if bits < 1 or bits > 8:
        raise InvalidInput("calibrate: bits must be in [1,8]")
    if scheme == Scheme.symmetric and bits < 2:
        raise InvalidInput("calibrate_symmetric: bits must be >= 2")
    if not np.all(np.isfinite(values)):
        raise InvalidInput("calibrate: non-finite value")
    cfg = QuantConfig(bits, scheme, Granularity.per_tensor, 0)
    return calibrate_grids(values.reshape(1, -1), cfg, mode)


def quantize_matrix(w: np.ndarray, cfg: QuantConfig, mode: ScaleMode = ScaleMode.minmax) -> QuantizedMatrix:
    """RTN quantize_matrix (quant.cpp:198-210)."""
    w = np.asarray(w, dtype=np.float32)
    grids = calibrate_grids(w, cfg, mode)
    gi = group_index_matrix(cfg, *w.shape)
    codes, _ = quantize_scalar(w, grids.scale[gi], grids.zero[gi], grids.qmin, grids.qmax)
    return QuantizedMatrix(w.shape[0], w.shape[1], cfg, codes.astype(np.int16), grids)


def dequantize(q: QuantizedMatrix) -> np.ndarray:
    """quant.cpp:212-218."""
    gi = group_index_matrix(q.config, q.rows, q.cols)
    return dequantize_scalar(q.codes.reshape(q.rows, q.cols), q.grids.scale[gi], q.grids.zero[gi])


def uniform_storage_bytes(cfg: QuantConfig, rows: int, cols: int) -> int:
    """quant.cpp:220-224."""
    code_bits = rows * cols * cfg.bits
    meta = 2 + (1 if cfg.scheme == Scheme.asymmetric else 0)
    return (code_bits + 7) // 8 + quant_group_count(cfg, rows, cols) * meta


def activation_objective(w, w_hat, h) -> float:
    """tr((W_hat - W)^T H (W_hat - W)) in fp64 (quant.cpp:230-236)."""
    w = np.asarray(w, dtype=np.float32)
    w_hat = np.asarray(w_hat, dtype=np.float32)
    h = np.asarray(h, dtype=np.float32)
    if w.shape != w_hat.shape:
        raise InvalidInput("activation_objective: shape mismatch")
    if h.shape[0] != h.shape[1] or h.shape[0] != w.shape[0]:
        raise InvalidInput("activation_objective: H must be N x N with N = rows of W")
    d = w_hat.astype(np.float64) - w.astype(np.float64)
    return float(np.einsum("ij,ij->", d, h.astype(np.float64) @ d))


# --------------------------------------------------------------------------
# calibration statistics (stats.cpp:10-19)
# --------------------------------------------------------------------------


@dataclass
class CalibStats:
    """stats.hpp:13-27: fp64 gram / cross, token count."""
    gram: np.ndarray
    cross: np.ndarray
    token_count: int = 0

    @staticmethod
    def zeros(dim: int) -> "CalibStats":
        return CalibStats(np.zeros((dim, dim)), np.zeros((dim, dim)), 0)

    def dim(self) -> int:
        return self.gram.shape[0]

    def gram_matrix(self) -> np.ndarray:
        """stats.cpp:7 -> eigen_map.hpp:25-29: fp64 -> fp32 cast."""
        return self.gram.astype(np.float32)


def accumulate_stats(stats: CalibStats, x_fp: np.ndarray, x_pert: np.ndarray) -> None:
    """gram += Xp^T Xp; cross += Xp^T (X - Xp), fp64 (stats.cpp:10-19)."""
    x_fp = np.asarray(x_fp, dtype=np.float32)
    x_pert = np.asarray(x_pert, dtype=np.float32)
    if x_fp.shape != x_pert.shape:
        raise InvalidInput("accumulate_stats: shape mismatch")
    if x_fp.shape[1] != stats.dim():
        raise InvalidInput("accumulate_stats: stats dimension does not match inputs")
    xp = x_pert.astype(np.float64)
    stats.gram += xp.T @ xp
    stats.cross += xp.T @ (x_fp.astype(np.float64) - xp)
    stats.token_count += x_fp.shape[0]


def gram_of_bf16_rows(x: np.ndarray, chunk: int = 8192) -> np.ndarray:
    """fp64 X^T X of a (T x N) matrix, streamed in token chunks (stats.cpp:16).

    Same arithmetic as accumulate_stats(stats, x, x) restricted to the gram
    (cross is identically 0 when x_fp == x_pert, test_core.cpp:273-279).
    """
    n = x.shape[1]
    g = np.zeros((n, n), dtype=np.float64)
    for t0 in range(0, x.shape[0], chunk):
        xc = np.asarray(x[t0:t0 + chunk], dtype=np.float64)
        g += xc.T @ xc
    return g


# --------------------------------------------------------------------------
# GPTQ (layerwise.cpp:11-93)
# --------------------------------------------------------------------------


@dataclass
class GptqOptions:
    """layerwise.hpp:11-15."""
    actorder: bool = False
    percdamp: float = 0.01
    block_cols: int = 32


def gptq_order(h: np.ndarray, actorder: bool) -> np.ndarray:
    """layerwise.cpp:11-18: stable sort by descending fp32 diag(H), ties by index."""
    n = h.shape[0]
    if not actorder:
        return np.arange(n, dtype=np.int64)
    d = np.asarray(np.diagonal(h), dtype=np.float32)
    # stable ascending sort of -d == stable descending sort of d (d >= 0 or NaN-free)
    return np.argsort(-d, kind="stable").astype(np.int64)


def _cholesky_lower(a: np.ndarray, what: str) -> np.ndarray:
    """Eigen::LLT<MatrixXd> (reads the lower triangle); numeric_error on breakdown."""
    import scipy.linalg as sla
    try:
        return sla.cholesky(np.tril(a) + np.tril(a, -1).T, lower=True, check_finite=False)
    except (np.linalg.LinAlgError, sla.LinAlgError):
        raise NumericError(what) from None


def gptq_factor(h: np.ndarray, order: np.ndarray, percdamp: float):
    """Damping, permutation, LLT, inverse, LLT (layerwise.cpp:31-51).

    Returns (U upper with hp^-1 = U^T U, hinv = hp^-1, damp), all fp64.
    """
    import scipy.linalg as sla
    hd = np.asarray(h, dtype=np.float32).astype(np.float64)
    damp = percdamp * float(np.mean(np.diagonal(hd)))
    hd[np.diag_indices_from(hd)] += damp
    hp = hd[np.ix_(order, order)]
    if not np.all(np.isfinite(hp)):
        raise NumericError("gptq_quantize: Gram matrix is not positive definite after dampening")
    L = _cholesky_lower(hp, "gptq_quantize: Gram matrix is not positive definite after dampening")
    n = hp.shape[0]
    hinv = sla.cho_solve((L, True), np.eye(n), check_finite=False)
    L2 = _cholesky_lower(hinv, "gptq_quantize: inverse Gram factorization failed")
    return L2.T.copy(), hinv, damp


def gptq_quantize(w: np.ndarray, h: np.ndarray, cfg: QuantConfig, opts: GptqOptions = GptqOptions(),
                  mode: ScaleMode = ScaleMode.minmax, return_debug: bool = False) -> QuantizedMatrix:
    """Hessian-aware sequential quantization, restating layerwise.cpp:20-93 in fp64."""
    cfg.validate()                                                           # :22
    w = np.asarray(w, dtype=np.float32)
    h = np.asarray(h, dtype=np.float32)
    if h.ndim != 2 or h.shape[0] != h.shape[1] or h.shape[0] != w.shape[0]:  # :23-24
        raise InvalidInput("gptq_quantize: H must be N x N with N = rows of W")
    if not (opts.percdamp > 0.0) or opts.percdamp > 1.0:                     # :25-26
        raise InvalidInput("gptq_quantize: percdamp must be in (0, 1]")
    n, m = w.shape
    order = gptq_order(h, opts.actorder)                                     # :29
    u, hinv, damp = gptq_factor(h, order, opts.percdamp)                     # :31-51
    grids = calibrate_grids(w, cfg, mode)                                    # :58-60
    gpr = quant_groups_per_row(cfg, m)
    if cfg.granularity == Granularity.per_tensor:
        gcols = np.zeros(m, dtype=np.int64)
    elif cfg.granularity == Granularity.per_channel:
        gcols = np.zeros(m, dtype=np.int64)
    else:
        gcols = np.arange(m, dtype=np.int64) // cfg.group_size

    def grid_row(orig):
        if cfg.granularity == Granularity.per_tensor:
            return np.zeros(m, dtype=np.int64)
        if cfg.granularity == Granularity.per_channel:
            return np.full(m, orig, dtype=np.int64)
        return orig * gpr + gcols

    wp = w[order].astype(np.float64)                                         # :40
    codes = np.zeros((n, m), dtype=np.int16)
    block = max(1, int(opts.block_cols))                                     # :62
    for ib in range(0, n, block):                                            # :65
        ie = min(n, ib + block)
        err = np.zeros((ie - ib, m), dtype=np.float64)
        for i in range(ib, ie):                                              # :68
            orig = int(order[i])
            row_f = wp[i].astype(np.float32)                                 # :70
            d = u[i, i]                                                      # :72
            g = grid_row(orig)
            code, w_hat = quantize_scalar(row_f, grids.scale[g], grids.zero[g], grids.qmin, grids.qmax)
            codes[orig] = code.astype(np.int16)                              # :75
            err[i - ib] = (wp[i] - w_hat.astype(np.float64)) / d             # :76-77
            if i + 1 < ie:                                                   # :80-82
                wp[i + 1:ie] -= np.outer(u[i, i + 1:ie], err[i - ib])
        if ie < n:                                                           # :85-90
            wp[ie:] -= u[ib:ie, ie:].T @ err
    q = QuantizedMatrix(n, m, cfg, codes, grids)
    if return_debug:
        q.extra = {"order": order, "u": u, "hinv": hinv, "damp": damp}
    return q


@dataclass
class LayerQuantOptions:
    """layerwise.hpp:41-47 (QEP omitted: next-row f1)."""
    method: str = "gptq"
    config: QuantConfig = field(default_factory=QuantConfig)
    scale_mode: ScaleMode = ScaleMode.minmax
    gptq: GptqOptions = field(default_factory=GptqOptions)


def quantize_layer(w: np.ndarray, stats: CalibStats, opts: LayerQuantOptions) -> QuantizedMatrix:
    """layerwise.cpp:120-126 without QEP."""
    if opts.method == "rtn":
        return quantize_matrix(w, opts.config, opts.scale_mode)
    return gptq_quantize(w, stats.gram_matrix(), opts.config, opts.gptq, opts.scale_mode)


# --------------------------------------------------------------------------
# OCW1 uniform payload (container.cpp:15-35 BitWriter, 66-70 put_fp16,
# 129-139 payload, 168-199 parse)
# --------------------------------------------------------------------------


def pack_uniform(codes: np.ndarray, grids: Grids, cfg: QuantConfig) -> bytes:
    """Codes (c - qmin) in b bits, one continuous LSB-first stream, one final
    flush; then fp16 LE scales in group order; then u8 zeros if asymmetric."""
    b = cfg.bits
    qmin = scheme_qmin(b, cfg.scheme)
    v = (np.asarray(codes, dtype=np.int64).ravel() - qmin).astype(np.uint32)
    bits = ((v[:, None] >> np.arange(b, dtype=np.uint32)[None, :]) & 1).astype(np.uint8).ravel()
    code_bytes = np.packbits(bits, bitorder="little").tobytes()
    sc = fp16_encode(grids.scale).astype("<u2").tobytes()
    out = code_bytes + sc
    if cfg.scheme == Scheme.asymmetric:
        out += (np.asarray(grids.zero, dtype=np.int64) & 0xFF).astype(np.uint8).tobytes()
    return out


def unpack_uniform(payload: bytes, rows: int, cols: int, cfg: QuantConfig) -> QuantizedMatrix:
    """container.cpp:168-199."""
    b = cfg.bits
    qmin, qmax = scheme_qmin(b, cfg.scheme), scheme_qmax(b, cfg.scheme)
    n_codes = rows * cols
    code_bytes = (n_codes * b + 7) // 8
    ng = quant_group_count(cfg, rows, cols)
    if len(payload) != uniform_storage_bytes(cfg, rows, cols):
        raise IOError("container: uniform payload size mismatch")
    raw = np.frombuffer(payload, dtype=np.uint8)
    bits = np.unpackbits(raw[:code_bytes], bitorder="little")[: n_codes * b].reshape(n_codes, b)
    v = (bits.astype(np.int64) << np.arange(b)[None, :]).sum(axis=1)
    codes = (v + qmin).astype(np.int16)
    sc = fp16_decode(np.frombuffer(payload[code_bytes:code_bytes + 2 * ng], dtype="<u2"))
    if cfg.scheme == Scheme.asymmetric:
        z = np.frombuffer(payload[code_bytes + 2 * ng:], dtype=np.uint8).astype(np.int32)
    else:
        z = np.zeros(ng, dtype=np.int32)
    return QuantizedMatrix(rows, cols, cfg, codes, Grids(sc.astype(np.float32), z, qmin, qmax))


# --------------------------------------------------------------------------
# reference fixtures (include/ocw/rng.hpp:12-57, matrix.cpp:57-62)
# --------------------------------------------------------------------------

_M64 = (1 << 64) - 1


class Rng:
    """splitmix64-seeded xorshift64* + Box-Muller, exactly rng.hpp:12-57."""

    def __init__(self, seed: int):
        z = (seed + 0x9E3779B97F4A7C15) & _M64
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        self.state = z ^ (z >> 31)
        if self.state == 0:
            self.state = 0x9E3779B97F4A7C15
        self.spare = 0.0
        self.has_spare = False

    def next_u64(self) -> int:
        x = self.state
        x ^= x >> 12
        x = (x ^ (x << 25)) & _M64
        x ^= x >> 27
        self.state = x
        return (x * 2685821657736338717) & _M64

    def uniform(self) -> float:
        return float(self.next_u64() >> 11) * 2.0**-53

    def below(self, n: int) -> int:
        return self.next_u64() % n if n else 0

    def gaussian(self) -> float:
        import math
        if self.has_spare:
            self.has_spare = False
            return self.spare
        u1, u2 = self.uniform(), self.uniform()
        while u1 <= 1e-300:
            u1 = self.uniform()
        r = math.sqrt(-2.0 * math.log(u1))
        theta = 2.0 * 3.14159265358979323846 * u2
        self.spare = r * math.sin(theta)
        self.has_spare = True
        return r * math.cos(theta)


def random_gaussian(rows: int, cols: int, seed: int, stddev: float = 1.0) -> np.ndarray:
    """matrix.cpp:57-62: float(rng.gaussian()) * stddev, row-major."""
    rng = Rng(seed)
    out = np.empty(rows * cols, dtype=np.float32)
    sd = np.float32(stddev)
    for k in range(rows * cols):
        out[k] = np.float32(rng.gaussian()) * sd
    return out.reshape(rows, cols)


def identity(n: int) -> np.ndarray:
    return np.eye(n, dtype=np.float32)


def bf16_round(x) -> np.ndarray:
    """fp32 -> nearest bf16 (ties-to-even) -> fp32; the BASELINE configs draw X
    this way ("each value rounded to bf16")."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).reshape(np.shape(x))


def bf16_bits(x) -> np.ndarray:
    """fp32 -> bf16 bit patterns (uint16), ties-to-even."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16).reshape(np.shape(x))
