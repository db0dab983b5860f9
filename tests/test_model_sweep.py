"""Host logic of the whole-model sweep (C4, paper_2603_28845_b200/model_sweep.py)
on CPU: the unit list mirrors the model's taps (model.cpp:301-307), LPT
assigns every unit exactly once with balanced loads, seeds are distinct, and
the payload gather brings every layer to rank 0 (gloo, 3 ranks)."""
import os
import socket

import pytest

from paper_2603_28845_b200 import model_sweep as MS


def test_units_cover_the_model():
    units = MS.model_units()
    assert len(units) == 128
    names = [n for u in units for n in MS.layer_names(u)]
    assert len(names) == 224 and len(set(names)) == 224
    weights = sum(u.n * m for u in units for _, m in u.linears)
    assert weights == 32 * (4 * 4096 * 4096 + 2 * 4096 * 11008 + 11008 * 4096)
    assert [u.tap for u in units[:4]] == ["attn_in", "o_in", "mlp_in", "down_in"]
    assert all(u.silu == (u.tap == "down_in") for u in units)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_lpt_plan(world):
    units = MS.model_units()
    plan = MS.lpt(units, world)
    assert len(plan) == world
    flat = [u for p in plan for u in p]
    assert sorted(flat, key=lambda u: u.index) == units  # every unit exactly once
    loads = [sum(MS.unit_cost(u) for u in p) for p in plan]
    biggest = max(MS.unit_cost(u) for u in units)
    assert max(loads) - min(loads) <= biggest + 1e-12  # LPT bound
    assert plan == MS.lpt(units, world)  # deterministic
    for p in plan:
        assert [u.index for u in p] == sorted(u.index for u in p)  # model order per rank


def test_down_unit_weighs_most():
    units = MS.model_units(1)
    c = {u.tap: MS.unit_cost(u) for u in units}
    assert c["down_in"] > 3 * c["attn_in"] > 3 * c["o_in"] / 2


def test_seeds_distinct():
    units = MS.model_units()
    xs = [MS.seeds(u)["x"] for u in units]
    ws = [s for u in units for s in MS.seeds(u)["w"]]
    assert len(set(xs)) == 128 and len(set(ws)) == 224


def _pb(n, m):
    return (n * m * 4 + 7) // 8 + (n * ((m + 127) // 128)) * 3


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        units = MS.model_units(2, hidden=64, ffn=192)  # small shapes, same structure
        plan = MS.lpt(units, world, tokens=1024)
        mine = {}
        for u in plan[rank]:
            for (name, m), key in zip(u.linears, MS.layer_names(u)):
                mine[key] = torch.full((_pb(u.n, m),), (sum(key.encode()) % 251), dtype=torch.uint8)
        out = MS.gather_payloads(plan, mine, _pb)
        if rank == 0:
            q.put({k: (int(v.numel()), int(v[0]), int(v[-1])) for k, v in out.items()})
        else:
            assert out is None
    finally:
        dist.destroy_process_group()


def test_gather_payloads_gloo():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    world = 3
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    units = MS.model_units(2, hidden=64, ffn=192)
    for u in units:
        for (name, m), key in zip(u.linears, MS.layer_names(u)):
            assert got[key] == (_pb(u.n, m), sum(key.encode()) % 251, sum(key.encode()) % 251)
