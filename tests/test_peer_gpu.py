"""Fused peer-memory gradient exchange (csrc/kernels/peer.cu): reduce 1/N of
the gradients from every rank over P2P, SGD, store the new weights into every
rank's arena -- checked against the host-side reduction of the same
gradients.

The driver's GPU box has one B200, so the multi-rank cases run N processes on
the SAME device: CUDA IPC maps each process's arenas into the others exactly
as across GPUs (only the link differs), and the flag barriers synchronise
separate contexts. Handles travel over gloo.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

LR = 0.05


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _session(V, numeric, g, cm, external=True):
    d = V.static_decision(V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal, g, cm)
    s = V.Session(g, d, cm, 64 << 20, external_grads=external)
    w = numeric.he_weights(g, cm, seed=31)
    for k, v in w.items():
        s.set_weights(k, v)
    return s, w


def _batch(g, seed):
    sh = g.shape(0)
    rng = np.random.default_rng(seed)
    images = rng.uniform(-1, 1, size=(sh.n, sh.h, sh.w, sh.c)).astype(np.float32)
    labels = rng.integers(0, 10, size=sh.n).astype(np.int32)
    return images, labels


@pytest.mark.parametrize("es", [4, 2], ids=["fp32", "bf16"])
def test_peer_exchange_world1_equals_apply_grads(es):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1602_08124_b200 as V
    from oracle import numeric
    g = V.build_preset("inception_toy", 8)
    cm = V.CostModel()
    cm.elem_size = es
    images, labels = _batch(g, 41)
    outs = []
    for peer in (False, True):
        s, w = _session(V, numeric, g, cm)
        s.set_batch(images, labels)
        if peer:
            s.peer_attach(0, [s.peer_export()])
            s.step(LR, want_loss=False)
            s.peer_exchange(LR, 1.0)
        else:
            s.step(LR, want_loss=False)
            s.apply_grads(LR, 1.0)
        s.synchronize()
        outs.append({k: s.get_weights(k) for k in w})
        if peer:
            s.peer_detach()
        del s
    for k in outs[0]:
        assert np.array_equal(outs[0][k], outs[1][k]), k  # same SGD expression, bit-identical


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        import paper_1602_08124_b200 as V
        from oracle import numeric
        from paper_1602_08124_b200.dist import PeerDataParallel
        g = V.build_preset("inception_toy", 8)
        cm = V.CostModel()
        s, w = _session(V, numeric, g, cm)
        dp = PeerDataParallel(s, world, overlap=False)  # the exchange after the step, checked in between
        report = []
        for it in range(2):
            images, labels = _batch(g, 100 + 10 * it + rank)
            s.set_batch(images, labels)
            w0 = {k: s.get_weights(k) for k in w}
            s.step(LR, want_loss=False)
            s.synchronize()
            grads = {k: s.get_grads(k) for k in w}
            all_grads = [None] * world
            dist.all_gather_object(all_grads, grads)
            s.peer_exchange(LR, 1.0 / world)
            s.synchronize()
            w1 = {k: s.get_weights(k) for k in w}
            all_w1 = [None] * world
            dist.all_gather_object(all_w1, w1)
            err = 0.0
            same = True
            for k in w:
                acc = all_grads[0][k].copy()
                for p in range(1, world):
                    acc = acc + all_grads[p][k]  # rank order, fp32
                # the kernel's step = float(lr) * float(1/N), then one fused
                # multiply-add w - step*sum: exact in float64, rounded once
                step = np.float32(np.float32(LR) * np.float32(1.0 / world))
                ref = (w0[k].astype(np.float64) - np.float64(step) * acc.astype(np.float64)).astype(np.float32)
                ulps = np.abs(w1[k] - ref) / np.spacing(np.maximum(np.abs(ref), np.float32(1e-30)))
                err = max(err, float(np.max(ulps)))
                same = same and all(np.array_equal(all_w1[p][k], w1[k]) for p in range(world))
            report.append((err, same))
        dp.close()
        q.put((rank, report, None))
        dist.destroy_process_group()
    except Exception as e:  # surfaced by the parent
        q.put((rank, None, repr(e)))


def _overlap_worker(rank, world, port, q, es=4):
    """Two sessions per rank over the same batches: the in-step exchange
    (each layer right after its wgrad, on a side stream) and the exchange after
    the step. Weights must be bit-identical between the two modes and across
    ranks after every step."""
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import hashlib
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        import paper_1602_08124_b200 as V
        from oracle import numeric
        from paper_1602_08124_b200.dist import PeerDataParallel
        g = V.build_preset("inception_toy", 8)
        cm = V.CostModel()
        cm.elem_size = es
        runs = {}
        for overlap in (True, False):
            s, w = _session(V, numeric, g, cm)
            dp = PeerDataParallel(s, world, overlap=overlap)
            digests, losses = [], []
            for it in range(3):
                images, labels = _batch(g, 300 + 10 * it + rank)
                s.set_batch(images, labels)
                losses.append(dp.step(LR, want_loss=True))
                s.synchronize()
                h = hashlib.sha256()
                for k in sorted(w):
                    h.update(s.get_weights(k).tobytes())
                digests.append(h.hexdigest())
            runs[overlap] = (digests, losses, dp.mode)
            dp.close()
            del s
        all_d = [None] * world
        dist.all_gather_object(all_d, runs[True][0])
        q.put((rank, {"same_modes": runs[True][0] == runs[False][0], "same_ranks": all(d == all_d[0] for d in all_d),
                      "losses_equal": runs[True][1] == runs[False][1], "mode": runs[True][2]}, None))
        dist.destroy_process_group()
    except Exception as e:
        q.put((rank, None, repr(e)))


@pytest.mark.parametrize("world,es", [(2, 4), (4, 4), (8, 4), (2, 2)], ids=["w2", "w4", "w8", "w2-bf16"])
def test_peer_exchange_inside_the_step_is_bit_identical(world, es):
    """SURVEY §8(e) placement at world 2, 4 and 8 (N processes sharing the
    box's one device through CUDA IPC); bf16 weights (elem_size 2) too."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_overlap_worker, args=(r, world, port, q, es)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
    for rank, rep, exc in res:
        assert exc is None, (rank, exc)
        assert rep["mode"] == "peer-overlap", rep
        assert rep["same_modes"] and rep["same_ranks"] and rep["losses_equal"], (rank, rep)


def _spill_worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        import paper_1602_08124_b200 as V
        from oracle import numeric
        from paper_1602_08124_b200.dist import PeerDataParallel, ring_spill
        g = V.build_preset("alexnet", 4)
        cm = V.CostModel()
        d = V.static_decision(V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal, g, cm)
        w = numeric.he_weights(g, cm, seed=51)
        images, labels = _batch(g, 60 + rank)
        labels = labels % 1000
        # data parallel, offloads into the ring neighbour's spill buffer
        s = V.Session(g, d, cm, 1 << 30, external_grads=True, offload_target="device", record_timeline=True)
        for k, v in w.items():
            s.set_weights(k, v)
        peer = ring_spill(s, world)
        dp = PeerDataParallel(s, world, overlap=False)
        s.set_batch(images, labels)
        s.step(LR, want_loss=False)
        s.synchronize()
        grads = {k: s.get_grads(k) for k in w}
        s.peer_exchange(LR, 1.0 / world)
        s.synchronize()
        after = {k: s.get_weights(k) for k in w}
        clean = V.replay_check(s.measured_report(), g, d, 1 << 30) == []
        dist.barrier()  # every rank done with its neighbour's spill buffer
        dp.close()
        del s
        # the same batch through the pinned host arena: identical gradients
        s2 = V.Session(g, d, cm, 1 << 30, external_grads=True)
        for k, v in w.items():
            s2.set_weights(k, v)
        s2.set_batch(images, labels)
        s2.step(LR, want_loss=False)
        s2.synchronize()
        same_grads = all(np.array_equal(s2.get_grads(k), grads[k]) for k in w)
        all_after = [None] * world
        dist.all_gather_object(all_after, after)
        same_w = all(np.array_equal(all_after[p][k], after[k]) for p in range(world) for k in w)
        q.put((rank, (peer, clean, same_grads, same_w), None))
        dist.destroy_process_group()
    except Exception as e:
        q.put((rank, None, repr(e)))


def test_ring_spill_offload_multiprocess_same_device():
    """Peer-HBM offload target: each rank offloads into its ring neighbour's
    spill buffer (CUDA IPC; over NVLink between GPUs), together with the
    fused gradient exchange. Gradients equal the pinned-host-arena run bit
    for bit, the measured log replays clean, and ranks end identical."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_spill_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
    for rank, rep, exc in res:
        assert exc is None, (rank, exc)
        peer, clean, same_grads, same_w = rep
        assert peer == (rank + 1) % world and clean and same_grads and same_w, (rank, rep)


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_peer_exchange_multiprocess_same_device(world):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
    for rank, report, exc in res:
        assert exc is None, (rank, exc)
        for err, same in report:
            assert err <= 1.0, (rank, err)  # within one ulp of the fused reference
            assert same, rank  # every rank holds bit-identical weights


def test_bench_two_ranks_same_device_peer_exchange():
    """bench.py's N>1 path end to end (torchrun, 2 ranks): on the one-GPU box
    both ranks share cuda:0 (VDNN_BENCH_SAME_DEVICE=1 -> gloo for the host
    collectives); the gradient exchange is the fused peer kernel, and the
    dynp policy offloads into the neighbour rank's spill buffer."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, VDNN_BENCH_SAME_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--net", "alexnet", "--batch", "32", "--policies", "dyn,dynp,none", "--steps", "1", "--warmup", "3",
           "--no-cpu-baseline"]
    out = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0
    assert line["config"]["gradient_exchange"] == "peer-overlap"
    assert line["policies"]["dyn"]["dp_exchange"] == "peer-overlap"
    census = line["rank_census"]
    assert [c["rank"] for c in census] == [0, 1] and all(c["exchange"] == "peer-overlap" for c in census)
    # the same plan offloading into the ring neighbour's HBM
    assert line["policies"]["dynp"]["signature"] == line["policies"]["dyn"]["signature"]
    assert line["peer_hbm_offload"]["images_per_s"] > 0


def test_bench_two_ranks_compressed_transfers_bit_identical():
    """N>1 with the compressed transfer modes (in bench.py's multi-GPU default
    policies): under a budget that makes vDNN_dyn offload, copy-engine,
    lossless-compressed and TF32-exact transfers give the same loss on 2 ranks
    with the fused peer gradient exchange."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, VDNN_BENCH_SAME_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--net", "alexnet", "--batch", "32", "--capacity", "271494988", "--policies", "dyn,dynz,dynt",
           "--steps", "1", "--warmup", "3", "--no-cpu-baseline"]
    out = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    pol = line["policies"]
    assert pol["dyn"]["offload_bytes_per_iter"] > 0
    assert pol["dyn"]["loss"] == pol["dynz"]["loss"] == pol["dynt"]["loss"]
    assert pol["dynt"]["wire_ratio"] < pol["dynz"]["wire_ratio"] < 1.0
