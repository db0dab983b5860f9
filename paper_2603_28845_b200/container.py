"""OCW1 container for the tensors this path produces.

Restates the reference's file format (src/container.cpp):
  "OCW1" | u64 LE header length | header JSON | payloads, in file order
(serialize_ocw :344-373).  The header is nlohmann::json's compact dump() of
  {"meta": <meta or {}>, "tensors": [{"bytes", "encoding", "name", "offset",
   ["params"], "shape"}, ...]}
with object keys in std::map (byte-wise) order.  Records:
  * uniform-quant (TensorRecord::from_uniform :278-289): params bits, scheme
    ("symmetric" / "asymmetric"), granularity ("per-tensor" / "per-channel" /
    "per-group"), group_size (per-group only); payload = the OCW1 uniform
    bitstream + fp16 scales + u8 zeros (tensor_payload :129-139) -- produced on
    the GPU by pack_uniform (or passed in, e.g. from quantize_layer_x);
  * f32 (from_f32 :270-276): little-endian fp32 values.
Parsing follows deserialize_ocw (:375-): magic, header bounds, per-tensor
payload bounds and size accounting, io_error on any mismatch; uniform payloads
are decoded on the GPU (unpack_uniform).

Byte-identity with the reference's serialize_ocw is checked in
tests/test_container.py against container.cpp itself (oracle/_ref).
"""
from __future__ import annotations

import json
import struct
from dataclasses import dataclass, field

import numpy as np

from . import (Granularity, InvalidInput, IoError, QuantConfig, QuantizedMatrix, Scheme,
               pack_uniform, uniform_storage_bytes, unpack_uniform)

MAGIC = b"OCW1"
_SCHEME = {Scheme.symmetric: "symmetric", Scheme.asymmetric: "asymmetric"}
_GRAN = {Granularity.per_tensor: "per-tensor", Granularity.per_channel: "per-channel",
         Granularity.per_group: "per-group"}


@dataclass
class Record:
    """One tensor of an OCW1 file (TensorRecord, container.hpp:44-62)."""
    name: str
    encoding: str                 # "uniform-quant" | "f32"
    shape: tuple
    params: dict = field(default_factory=dict)
    payload: bytes = b""
    value: object = None          # QuantizedMatrix or np.ndarray (decoded)


def uniform_record(name: str, q: QuantizedMatrix, payload: bytes | None = None) -> Record:
    """TensorRecord::from_uniform (container.cpp:278-289); the payload is
    packed on the GPU unless given (e.g. quantize_layer_x's)."""
    c = q.config
    params = {"bits": int(c.bits), "scheme": _SCHEME[Scheme(int(c.scheme))],
              "granularity": _GRAN[Granularity(int(c.granularity))]}
    if Granularity(int(c.granularity)) == Granularity.per_group:
        params["group_size"] = int(c.group_size)
    if payload is None:
        payload = pack_uniform(q)
    return Record(name, "uniform-quant", (int(q.rows), int(q.cols)), params, bytes(payload), q)


def f32_record(name: str, a) -> Record:
    """TensorRecord::from_f32 (container.cpp:270-276)."""
    a = np.ascontiguousarray(a, np.float32)
    if a.ndim != 2:
        raise InvalidInput("container: f32 tensors are 2-D")
    return Record(name, "f32", (int(a.shape[0]), int(a.shape[1])), {},
                  a.astype("<f4", copy=False).tobytes(), a)


def _expected_bytes(r: Record) -> int:
    rows, cols = r.shape
    if r.encoding == "f32":
        return rows * cols * 4
    return uniform_storage_bytes(_config(r.params), rows, cols)


def _config(params: dict) -> QuantConfig:
    try:
        scheme = {v: k for k, v in _SCHEME.items()}[params["scheme"]]
        gran = {v: k for k, v in _GRAN.items()}[params["granularity"]]
        return QuantConfig(int(params["bits"]), scheme, gran, int(params.get("group_size", 0)))
    except KeyError as e:
        raise IoError(f"container: bad uniform params ({e})") from None


def _dump(obj) -> bytes:
    """nlohmann::json::dump() for this schema: compact, keys in byte order."""
    try:
        return json.dumps(obj, separators=(",", ":"), sort_keys=True, ensure_ascii=False,
                          allow_nan=False).encode("utf-8")
    except ValueError as e:
        raise InvalidInput(f"container: meta is not serialisable ({e})") from None


def serialize_ocw(records, meta: dict | None = None) -> bytes:
    """serialize_ocw (container.cpp:344-373)."""
    tensors, payload = [], bytearray()
    for r in records:
        if len(r.payload) != _expected_bytes(r):
            raise IoError(f"container: payload accounting mismatch for {r.name}")
        entry = {"name": r.name, "encoding": r.encoding, "shape": list(r.shape),
                 "offset": len(payload), "bytes": len(r.payload)}
        if r.params:
            entry["params"] = r.params
        payload += r.payload
        tensors.append(entry)
    header = _dump({"meta": {} if meta is None else meta, "tensors": tensors})
    return MAGIC + struct.pack("<Q", len(header)) + header + bytes(payload)


def deserialize_ocw(data: bytes, decode: bool = True):
    """deserialize_ocw (container.cpp:375-): (meta, [Record]); with decode,
    Record.value holds the QuantizedMatrix (GPU unpack) or the f32 array."""
    data = bytes(data)
    if len(data) < 12 or data[:4] != MAGIC:
        raise IoError("container: bad magic (not an OCW1 file)")
    hlen = struct.unpack("<Q", data[4:12])[0]
    if 12 + hlen > len(data):
        raise IoError("container: truncated header")
    try:
        header = json.loads(data[12:12 + hlen].decode("utf-8"))
    except ValueError as e:
        raise IoError(f"container: bad header ({e})") from None
    body = data[12 + hlen:]
    out = []
    expected = 0
    for t in header.get("tensors", []):
        off, nb = int(t["offset"]), int(t["bytes"])
        if off != expected:  # container.cpp:404
            raise IoError("container: tensor offsets must be ascending and packed")
        if off + nb > len(body):
            raise IoError("container: tensor exceeds payload")
        r = Record(t["name"], t["encoding"], tuple(int(v) for v in t["shape"]),
                   t.get("params", {}), body[off:off + nb])
        if r.encoding not in ("f32", "uniform-quant"):
            raise IoError(f"container: encoding {r.encoding} is outside this path")
        if len(r.payload) != _expected_bytes(r):
            raise IoError(f"container: payload size mismatch for {r.name}")
        if decode:
            rows, cols = r.shape
            if r.encoding == "f32":
                r.value = np.frombuffer(r.payload, "<f4").astype(np.float32).reshape(rows, cols)
            else:
                r.value = unpack_uniform(r.payload, rows, cols, _config(r.params))
        out.append(r)
        expected = off + nb
    if expected != len(body):  # container.cpp:411
        raise IoError("container: payload length does not match tensor sizes")
    return header.get("meta", {}), out


def store_ocw(path, records, meta: dict | None = None) -> None:
    """store_ocw (container.hpp:75)."""
    with open(path, "wb") as f:
        f.write(serialize_ocw(records, meta))


def load_ocw(path, decode: bool = True):
    """load_ocw (container.hpp:76)."""
    with open(path, "rb") as f:
        return deserialize_ocw(f.read(), decode)
