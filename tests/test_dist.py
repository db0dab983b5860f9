"""Host logic of the multi-GPU path (paper_2603_28845_b200/dist.py) on CPU:
token shards + one all-reduce + column slabs + per-row assembly, run as two
gloo ranks with the CPU oracle standing in for each rank's GPU compute.  The
assembled codes / grids / payload must equal the single-process result on the
same H bit for bit (columns are independent given H, layerwise.cpp:65-91)."""
import os
import socket

import numpy as np
import pytest

from paper_2603_28845_b200 import dist as D


def test_token_range_partitions():
    for t, w in [(10, 3), (262144, 8), (5, 5), (7, 2)]:
        spans = [D.token_range(t, r, w) for r in range(w)]
        assert spans[0][0] == 0 and spans[-1][1] == t
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1


def test_column_slabs_group_aligned():
    # C2: 32 groups of 128 -> 4 per rank at 8 ranks; C3 up: 86 groups of 128
    assert D.column_slabs(4096, 128, 4, 8) == [(i * 512, (i + 1) * 512) for i in range(8)]
    s = D.column_slabs(11008, 128, 3, 8)
    assert [ (b - a) // 128 for a, b in s] == [11, 11, 11, 11, 11, 11, 10, 10]
    assert s[-1][1] == 11008 and all(a % 128 == 0 for a, _ in s)
    with pytest.raises(ValueError):
        D.column_slabs(100, 5, 3, 2)  # 15 bits per group row: not byte aligned


class OracleOps:
    """Each rank's compute done by the numpy oracle (test stand-in for the GPU)."""

    def __init__(self, orc):
        self.orc = orc

    def gram(self, x_local):
        import torch
        return torch.from_numpy(x_local.astype(np.float64).T @ x_local.astype(np.float64))

    def gptq_slab(self, w, j0, j1, h, cfg, opts):
        import torch
        orc = self.orc
        hf = h.numpy().astype(np.float32)
        q = orc.gptq_quantize(w[:, j0:j1], hf, cfg, opts)
        wh = orc.dequantize(q)
        t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dt))  # noqa: E731
        payload = torch.frombuffer(bytearray(orc.pack_uniform(q.codes, q.grids, cfg)), dtype=torch.uint8)
        return D.SlabResult(j0, j1, t(q.codes, np.int16), t(q.grids.scale, np.float32),
                            t(q.grids.zero, np.int32), t(wh, np.float32), payload)


def _problem(orc):
    rng = np.random.default_rng(11)
    n, m, t = 24, 64, 200
    x = orc.bf16_round(rng.standard_normal((t, n)).astype(np.float32))
    w = (0.02 * rng.standard_normal((n, m))).astype(np.float32)
    cfg = orc.QuantConfig(4, orc.Scheme.asymmetric, orc.Granularity.per_group, 16)
    opts = orc.GptqOptions(True, 0.01, 8)
    return w, x, cfg, opts


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from oracle import ocw_oracle as orc
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w, x, cfg, opts = _problem(orc)
        t0, t1 = D.token_range(x.shape[0], rank, world)
        out = D.quantize_layer_sharded(w, x[t0:t1], x.shape[0], cfg, opts, ops=OracleOps(orc))
        if rank == 0:
            codes, scales, zeros, w_hat, payload = out
            q.put((codes.numpy(), scales.numpy(), zeros.numpy(), w_hat.numpy(),
                   payload.numpy().tobytes()))
        else:
            assert out is None
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_layer_matches_single_process(orc, world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    codes, scales, zeros, w_hat, payload = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single process, same H (sum of the two token-shard Grams, as the all-reduce forms it)
    w, x, cfg, opts = _problem(orc)
    h = sum(x[a:b].astype(np.float64).T @ x[a:b].astype(np.float64)
            for a, b in (D.token_range(x.shape[0], r, world) for r in range(world)))
    ref = orc.gptq_quantize(w, h.astype(np.float32), cfg, opts)
    np.testing.assert_array_equal(codes, ref.codes)
    np.testing.assert_array_equal(scales, ref.grids.scale)
    np.testing.assert_array_equal(zeros, ref.grids.zero)
    np.testing.assert_array_equal(w_hat, orc.dequantize(ref))
    assert payload == orc.pack_uniform(ref.codes, ref.grids, cfg)
