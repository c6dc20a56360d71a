"""Data-parallel training over NCCL: one process per GPU, each rank running its
own vDNN plan (identical per-rank schedule, weak scaling), weight gradients
averaged with one bucketed all-reduce over the session's gradient arena.

The reference has no multi-GPU path; BASELINE.json's config 5
(VGG-416 b32 per GPU at 2/4/8 GPUs) asks for this one exchange step. The
gradient arena is a torch-allocated device buffer handed to the session
(vdnn_session_set_grad_arena), so the all-reduce runs on the session's compute
stream with no extra copy.
"""
from __future__ import annotations

import os
from typing import Optional, Tuple


def env_rank() -> Tuple[int, int, int]:
    """(rank, local_rank, world_size) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


def allreduce_mean_(t, world: int, group=None) -> None:
    """In-place mean over ranks (sum all-reduce, then scale)."""
    import torch.distributed as dist
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        t.div_(world)


def max_over_ranks(value: float, world: int, device=None) -> float:
    """Max of a per-rank scalar (timings are reported as the slowest rank)."""
    if world <= 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class DataParallel:
    """Wraps a Session created with external_grads=True."""

    def __init__(self, session, world: int, device: int, group=None):
        import torch
        self.s = session
        self.world = world
        self.group = group
        _, count = session.grad_arena()
        self.grads = torch.zeros(max(count, 1), dtype=torch.float32, device=f"cuda:{device}")
        session.set_grad_arena(self.grads.data_ptr(), count)
        self.stream = torch.cuda.ExternalStream(session.stream, device=f"cuda:{device}")

    def step(self, lr: float, want_loss: bool = False) -> Optional[float]:
        import torch
        import torch.distributed as dist
        loss = self.s.step(lr, want_loss=want_loss)  # dW -> gradient arena (no local SGD)
        if self.world > 1:
            with torch.cuda.stream(self.stream):
                dist.all_reduce(self.grads, op=dist.ReduceOp.SUM, group=self.group)
        self.s.apply_grads(lr, 1.0 / self.world)
        return loss
