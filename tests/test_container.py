"""OCW1 container against the reference's own container.cpp
(compiled unmodified into oracle/_ref/libocw_ref_container.so with the
nlohmann/json 3.11.3 header the image ships).

CPU: the product's serializer on oracle-packed payloads (the GPU packer is
bit-exact with them, tests/test_gpu_parity.py::test_pack_unpack_exhaustive) must
produce the reference's bytes, and the reference's parser must reproduce our
files.  GPU: the same with the payloads packed / unpacked on the device."""
import json

import numpy as np
import pytest

from oracle import ref


def _need_container():
    if ref.container_lib() is None:
        pytest.skip("reference container.cpp not built (no nlohmann/json in this image)")


def _cases(orc):
    w1 = ref.random_gaussian(37, 300, 11, 0.02)
    w2 = ref.random_gaussian(16, 77, 12, 0.05)
    w3 = ref.random_gaussian(9, 40, 13)
    cfgs = [orc.QuantConfig(4, orc.Scheme.asymmetric, orc.Granularity.per_group, 128),
            orc.QuantConfig(3, orc.Scheme.symmetric, orc.Granularity.per_channel, 0),
            orc.QuantConfig(8, orc.Scheme.asymmetric, orc.Granularity.per_tensor, 0)]
    return [(f"layers.{i}.w", w, c) for i, (w, c) in enumerate(zip((w1, w2, w3), cfgs))]


def _records(g, orc, with_payload=True):
    from paper_2603_28845_b200 import container as ct
    recs, rrecs = [], []
    for name, w, c in _cases(orc):
        q = orc.quantize_matrix(w, c)
        gq = g.QuantizedMatrix(q.rows, q.cols, g.QuantConfig(c.bits, g.Scheme(int(c.scheme)),
                               g.Granularity(int(c.granularity)), c.group_size),
                               q.codes, q.grids.scale, q.grids.zero)
        pay = orc.pack_uniform(q.codes, q.grids, c) if with_payload else None
        recs.append(ct.uniform_record(name, gq, pay))
        rrecs.append(("uniform", name, q.codes, q.grids.scale, q.grids.zero, c.bits,
                      int(c.scheme), int(c.granularity), c.group_size))
    emb = ref.random_gaussian(5, 7, 3)
    recs.append(ct.f32_record("embed", emb))
    rrecs.append(("f32", "embed", emb))
    return recs, rrecs


META = {"model": "llama-2-7b-shaped", "layers": 32, "bpw": 4.25, "quantizer": "gptq",
        "notes": "tab\tquote\" unicode é", "flags": [True, False, None]}


def test_serialize_matches_reference(orc):
    import paper_2603_28845_b200 as g
    from paper_2603_28845_b200 import container as ct
    _need_container()
    recs, rrecs = _records(g, orc)
    ours = ct.serialize_ocw(recs, META)
    theirs = ref.serialize_ocw(rrecs, json.dumps(META))
    assert ours == theirs
    assert ref.roundtrip_ocw(ours) == ours  # the reference's parser reproduces our file
    assert ct.serialize_ocw(recs, META) == ours  # deterministic (test_pipeline.cpp:225-250)
    assert ct.serialize_ocw(recs) == ref.serialize_ocw(rrecs, None)  # meta defaults to {}


def test_parse_structure_and_errors(orc):
    import paper_2603_28845_b200 as g
    from paper_2603_28845_b200 import container as ct
    recs, _ = _records(g, orc)
    data = ct.serialize_ocw(recs, META)
    meta, back = ct.deserialize_ocw(data, decode=False)
    assert meta == json.loads(json.dumps(META))
    assert [r.name for r in back] == [r.name for r in recs]
    assert all(a.payload == b.payload and a.shape == b.shape and a.params == b.params
               for a, b in zip(back, recs))
    with pytest.raises(g.IoError):
        ct.deserialize_ocw(b"OCW2" + data[4:], decode=False)
    with pytest.raises(g.IoError):
        ct.deserialize_ocw(data[:40], decode=False)
    with pytest.raises(g.IoError):
        ct.deserialize_ocw(data[:-1], decode=False)
    bad = ct.Record("x", "uniform-quant", (4, 4), recs[0].params, b"\x00")
    with pytest.raises(g.IoError):
        ct.serialize_ocw([bad])
    # payload longer than the tensors account for (container.cpp:411)
    with pytest.raises(g.IoError, match="payload length"):
        ct.deserialize_ocw(data + b"\x00", decode=False)
    # offsets not ascending-and-packed (container.cpp:404): swap two entries' offsets
    import struct
    hlen = struct.unpack("<Q", data[4:12])[0]
    header = json.loads(data[12:12 + hlen])
    t = header["tensors"]
    t[0]["offset"], t[1]["offset"] = t[1]["offset"], t[0]["offset"]
    h2 = json.dumps(header, separators=(",", ":"), sort_keys=True).encode()
    with pytest.raises(g.IoError, match="ascending and packed"):
        ct.deserialize_ocw(b"OCW1" + struct.pack("<Q", len(h2)) + h2 + data[12 + hlen:], decode=False)


@pytest.mark.gpu
def test_gpu_pack_container_roundtrip(orc):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2603_28845_b200 as g
    from paper_2603_28845_b200 import container as ct
    _need_container()
    recs, rrecs = _records(g, orc, with_payload=False)  # payloads packed on the GPU
    data = ct.serialize_ocw(recs, META)
    assert data == ref.serialize_ocw(rrecs, json.dumps(META))
    _, back = ct.deserialize_ocw(data)  # payloads unpacked on the GPU
    for r, b in zip(recs, back):
        if r.encoding == "f32":
            np.testing.assert_array_equal(b.value, r.value)
        else:
            np.testing.assert_array_equal(b.value.codes, r.value.codes)
            np.testing.assert_array_equal(b.value.scales, r.value.scales)
            np.testing.assert_array_equal(b.value.zeros, r.value.zeros)
