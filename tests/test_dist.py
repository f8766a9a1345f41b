"""Host-side multi-process logic on CPU (gloo, world size 2).

* batch sharding: weak shards are disjoint and keep global image ids; balanced shards
  partition a fixed batch with the same looks mix on every rank;
* the timing reductions (max / sum over ranks) and the byte broadcast of the NCCL id;
* the row-slab ring: slab ranges, neighbours, and the ghost-row exchange plan exported by
  libfoe (foe_slab_exchange_plan: the order the C code posts its NCCL calls) replayed with gloo
  point-to-point messages: every rank's ghost rows equal the periodic neighbours' boundary rows,
  for 2 ranks (both neighbours are the same peer) and 4;
* the band gather: per-band partials all-gathered in rank order are the scene's band order.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_1404_5344_b200 import dist as D  # noqa: E402

HALO = 6


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange(slab: np.ndarray, rank: int, ws: int):
    """Ghost rows by the plan libfoe itself posts (foe_slab_exchange_plan, the C code's exchange
    order), replayed with gloo isend/irecv."""
    import paper_1404_5344_b200 as P
    bufs = {P.FOE_HALO_TOP_ROWS: torch.as_tensor(slab[:HALO].copy()),
            P.FOE_HALO_BOTTOM_ROWS: torch.as_tensor(slab[-HALO:].copy()),
            P.FOE_HALO_TOP_GHOST: torch.empty(HALO, slab.shape[1], dtype=torch.float64),
            P.FOE_HALO_BOTTOM_GHOST: torch.empty(HALO, slab.shape[1], dtype=torch.float64)}
    reqs = []
    for op, peer, buf in P.foe_slab_exchange_plan(ws, rank):
        if op == P.FOE_HALO_SEND:
            reqs.append(dist.isend(bufs[buf], dst=peer))
        else:
            reqs.append(dist.irecv(bufs[buf], src=peer))
    for r in reqs:
        r.wait()
    return bufs[P.FOE_HALO_TOP_GHOST].numpy(), bufs[P.FOE_HALO_BOTTOM_GHOST].numpy()


def _worker(rank, ws, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws),
                          LOCAL_RANK=str(rank))
        r, w, _ = D.init_process_group("gloo")
        assert (r, w) == (rank, ws)
        out = {}
        # batch shards
        out["weak"] = D.weak_shard(8, rank)
        looks = [1, 3, 8] * 5 + [1]
        out["balanced"] = D.balanced_shard(looks, rank, ws)
        # reductions
        out["max"] = D.max_over_ranks(float(rank + 1))
        out["sum"] = D.sum_over_ranks(float(rank + 1))
        out["id"] = D.share_bytes(bytes(range(128)) if rank == 0 else None)
        out["all_true"] = (D.all_true(True), D.all_true(rank == 0))
        # slab ring on a 256 x 40 scene
        H, W = 256, 40
        scene = np.arange(H * W, dtype=np.float64).reshape(H, W)
        r0, r1 = D.slab_rows(H, ws, rank)
        top, bot = _exchange(scene[r0:r1], rank, ws)
        out["ghost_ok"] = bool(np.array_equal(top, scene[np.arange(r0 - HALO, r0) % H]) and
                               np.array_equal(bot, scene[np.arange(r1, r1 + HALO) % H]))
        # band gather: partial of band k = k (global band index)
        nb = (r1 - r0) // 64
        mine = torch.arange(r0 // 64, r0 // 64 + nb, dtype=torch.float64)
        allb = [torch.empty(nb, dtype=torch.float64) for _ in range(ws)]
        dist.all_gather(allb, mine)
        out["bands"] = torch.cat(allb).tolist()
        D.barrier()
        q.put((rank, out))
        dist.destroy_process_group()
    except Exception as e:  # surface the failure in the parent
        q.put((rank, {"error": repr(e)}))


def _run(ws):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(ws))
    for p in ps:
        p.join(timeout=60)
    for r in range(ws):
        assert "error" not in res[r], res[r]
    return res


@pytest.fixture(scope="module")
def two_ranks():
    return _run(2)


def test_weak_and_balanced_shards(two_ranks):
    r = two_ranks
    assert r[0]["weak"] == list(range(8)) and r[1]["weak"] == list(range(8, 16))
    b0, b1 = set(r[0]["balanced"]), set(r[1]["balanced"])
    assert not (b0 & b1) and (b0 | b1) == set(range(16))
    looks = [1, 3, 8] * 5 + [1]
    for L in (1, 3, 8):
        c0 = sum(looks[i] == L for i in b0); c1 = sum(looks[i] == L for i in b1)
        assert abs(c0 - c1) <= 1


def test_reductions_and_id_broadcast(two_ranks):
    for rank in (0, 1):
        assert two_ranks[rank]["max"] == 2.0
        assert two_ranks[rank]["sum"] == 3.0
        assert two_ranks[rank]["id"] == bytes(range(128))
        assert two_ranks[rank]["all_true"] == (True, False)


def test_slab_ring_ghost_rows_two_ranks(two_ranks):
    assert two_ranks[0]["ghost_ok"] and two_ranks[1]["ghost_ok"]


def test_band_gather_is_scene_order(two_ranks):
    for rank in (0, 1):
        assert two_ranks[rank]["bands"] == [0.0, 1.0, 2.0, 3.0]


def test_slab_ring_four_ranks():
    """4 ranks: one 64-row band each, distinct up/down peers (gloo has no self-send: the
    1-rank ring is covered by the NCCL self-ring test on the GPU, tests/test_slabs.py)."""
    r = _run(4)
    for rank in range(4):
        assert r[rank]["ghost_ok"] and r[rank]["bands"] == [0.0, 1.0, 2.0, 3.0]
        assert r[rank]["max"] == 4.0 and r[rank]["sum"] == 10.0


def test_exchange_plan_is_the_ring_order():
    """The exported plan: send up, recv down, send down, recv up, peers on the periodic ring."""
    import paper_1404_5344_b200 as P
    for ws, rank in ((1, 0), (2, 0), (2, 1), (8, 0), (8, 7)):
        up, dn = D.ring_neighbours(rank, ws)
        assert P.foe_slab_exchange_plan(ws, rank) == [
            (P.FOE_HALO_SEND, up, P.FOE_HALO_TOP_ROWS), (P.FOE_HALO_RECV, dn, P.FOE_HALO_BOTTOM_GHOST),
            (P.FOE_HALO_SEND, dn, P.FOE_HALO_BOTTOM_ROWS), (P.FOE_HALO_RECV, up, P.FOE_HALO_TOP_GHOST)]
    with pytest.raises(P.FoeError):
        P.foe_slab_exchange_plan(2, 2)


def test_slab_geometry():
    assert D.slab_rows(8192, 8, 3) == (3072, 4096)
    assert D.ring_neighbours(0, 8) == (7, 1) and D.ring_neighbours(7, 8) == (6, 0)
    with pytest.raises(ValueError):
        D.slab_rows(8192 + 64, 8, 0)
