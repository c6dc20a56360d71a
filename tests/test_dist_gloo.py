"""Host-side logic of the data-parallel path on CPU (gloo, world_size 2):
gradient averaging and max-over-ranks timing used by bench.py."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1602_08124_b200.dist import allreduce_mean_, max_over_ranks
    g = torch.full((1000,), float(rank + 1))
    allreduce_mean_(g, world)
    t = max_over_ranks(10.0 + rank, world)
    q.put((rank, float(g[0]), float(g[-1]), t))
    dist.destroy_process_group()


def test_allreduce_mean_and_max_over_ranks():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    assert [r[1] for r in res] == [1.5, 1.5] and [r[2] for r in res] == [1.5, 1.5]
    assert [r[3] for r in res] == [11.0, 11.0]


def test_env_rank_defaults(monkeypatch):
    from paper_1602_08124_b200.dist import env_rank
    for k in ("RANK", "LOCAL_RANK", "WORLD_SIZE"):
        monkeypatch.delenv(k, raising=False)
    assert env_rank() == (0, 0, 1)


def test_make_data_parallel_rejects_unknown_mode():
    from paper_1602_08124_b200.dist import make_data_parallel
    with pytest.raises(ValueError):
        make_data_parallel(None, 2, 0, mode="ring")


class _FakeSession:
    """Stands in for Session in the host-side peer-attach protocol."""

    def __init__(self, rank, fail_rank):
        self.rank, self.fail_rank = rank, fail_rank
        self.attached = None
        self.detached = False

    def peer_export(self):
        return bytes([self.rank]) * 8

    def peer_attach(self, rank, handles):
        if rank == self.fail_rank:
            raise RuntimeError("cudaIpcOpenMemHandle refused")
        self.attached = (rank, list(handles))

    def peer_detach(self):
        self.detached = True

    def peer_overlap(self, on, scale):
        self.overlap = (on, scale)


def _peer_worker(rank, world, port, fail_rank, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1602_08124_b200.dist import PeerDataParallel, PeerUnavailable
    s = _FakeSession(rank, fail_rank)
    try:
        PeerDataParallel(s, world)
        q.put((rank, "ok", s.attached, s.detached))
    except PeerUnavailable as e:
        q.put((rank, "unavailable:" + str(e), s.attached, s.detached))
    dist.destroy_process_group()


@pytest.mark.parametrize("fail_rank", [-1, 1])
def test_peer_attach_all_or_none(fail_rank):
    """Handles are all-gathered in rank order; if any rank fails to attach,
    every rank detaches and raises (nobody is left waiting in a barrier)."""
    world = 3
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_peer_worker, args=(r, world, port, fail_rank, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    for rank, status, attached, detached in res:
        if fail_rank < 0:
            assert status == "ok" and attached == (rank, [bytes([r]) * 8 for r in range(world)]) and not detached
        else:
            assert status.startswith("unavailable:") and "rank 1" in status and detached


class _FakeSpillSession:
    def __init__(self, rank):
        self.rank = rank
        self.attached = None

    def spill_export(self):
        return bytes([0xA0 + self.rank]) * 64

    def spill_attach(self, handle):
        self.attached = handle


def _spill_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1602_08124_b200.dist import ring_spill
    s = _FakeSpillSession(rank)
    peer = ring_spill(s, world)
    q.put((rank, peer, s.attached))
    dist.destroy_process_group()


def test_ring_spill_routes_each_rank_to_its_neighbour():
    """Peer-HBM offload target: rank r offloads into rank (r+1) % N's spill
    buffer (the handle it attaches is the neighbour's export)."""
    world = 3
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_spill_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    for rank, peer, attached in res:
        assert peer == (rank + 1) % world
        assert attached == bytes([0xA0 + peer]) * 64


def test_ring_spill_needs_two_ranks():
    from paper_1602_08124_b200.dist import ring_spill
    with pytest.raises(ValueError):
        ring_spill(_FakeSpillSession(0), 1)
