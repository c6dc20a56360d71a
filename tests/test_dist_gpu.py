"""Data-parallel path on the GPU (world size 1 over NCCL): the gradient arena
is a torch tensor handed to the session, the all-reduce runs on the session
stream, apply_grads does the SGD -- and the result equals the fused path."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1602_08124_b200 as V
from oracle import numeric

pytestmark = pytest.mark.gpu


def test_dataparallel_world1_equals_fused_sgd():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.distributed as dist
    from paper_1602_08124_b200.dist import DataParallel
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        g = V.build_preset("alexnet", 4)
        cm = V.CostModel()
        d = V.static_decision(V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal, g, cm)
        w = numeric.he_weights(g, cm, seed=21)
        rng = np.random.default_rng(22)
        images = rng.uniform(-1, 1, size=(4, 227, 227, 3)).astype(np.float32)
        labels = rng.integers(0, 1000, size=4).astype(np.int32)
        outs = []
        for use_dp in (False, True):
            sess = V.Session(g, d, cm, 4 << 30, external_grads=use_dp)
            for k, v in w.items():
                sess.set_weights(k, v)
            sess.set_batch(images, labels)
            if use_dp:
                dp = DataParallel(sess, 1, 0)
                loss = dp.step(0.01, want_loss=True)
            else:
                loss = sess.step(0.01)
            outs.append((loss, {k: sess.get_weights(k) for k in w}))
        assert outs[0][0] == outs[1][0]
        for k in w:
            np.testing.assert_allclose(outs[1][1][k], outs[0][1][k], rtol=0, atol=1e-7)
    finally:
        dist.destroy_process_group()
