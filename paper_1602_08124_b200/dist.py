"""Data-parallel training: one process per GPU, each rank running its own vDNN
plan (identical per-rank schedule, weak scaling). Two exchange paths:

* ``PeerDataParallel`` (default): the fused peer-memory exchange of
  ``csrc/kernels/peer.cu`` -- every rank's arenas are mapped into every other
  rank through CUDA IPC; one kernel per rank reduces its 1/N share of the
  gradients from all ranks over NVLink, applies SGD and stores the new weights
  into every rank's arena (reduce-scatter + update + all-gather in one pass,
  bracketed by flag barriers). By default (overlap=True) each
  layer's share runs inside the step on a side stream right after that
  layer's wgrad, overlapping the rest of the backward pass; the step ends
  with one barrier. torch.distributed only carries the handles.
* ``DataParallel``: one bucketed NCCL all-reduce over the session's gradient
  arena followed by the SGD kernels (the library baseline).

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
    if dist.get_backend() == "gloo":
        device = "cpu"
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def make_data_parallel(session, world: int, device: int, mode: Optional[str] = None, group=None):
    """The exchange path for ``world`` ranks: ``mode`` "peer" (fused P2P
    kernel), "nccl", or None = $VDNN_DP, default "peer"."""
    mode = mode or os.environ.get("VDNN_DP", "peer")
    if mode == "peer":
        try:
            return PeerDataParallel(session, world, group=group)
        except PeerUnavailable as e:  # every rank agreed to fall back (no P2P between these GPUs)
            import sys
            print(f"[vdnn] peer exchange unavailable ({e}); using NCCL all-reduce", file=sys.stderr)
            mode = "nccl"
    if mode == "nccl":
        return DataParallel(session, world, device, group=group)
    raise ValueError(f"unknown data-parallel mode {mode!r}")


def bind_numa(device: int) -> Optional[str]:
    """Bind this process to the CPUs next to ``device`` (NVML's ideal affinity)
    before the session allocates its pinned host arena, so the arena's pages
    are first touched on the GPU's NUMA node (up to 64 GB per rank for
    VGG-416 b32 dyn). Returns the CPU list, or None if NVML is unavailable."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(device)
        pynvml.nvmlDeviceSetCpuAffinity(h)
        cpus = sorted(os.sched_getaffinity(0))
        return f"{cpus[0]}-{cpus[-1]} ({len(cpus)} cpus)" if cpus else None
    except Exception:
        return None


def rank_census(world: int, device: int, exchange: Optional[str], numa: Optional[str], group=None):
    """Every rank's (rank, device, GPU UUID, PCI bus id, exchange path, NUMA
    binding), gathered on all ranks: proof the N ranks ran on N devices."""
    import torch
    import torch.distributed as dist
    props = torch.cuda.get_device_properties(device)
    me = {"rank": dist.get_rank(group) if world > 1 else 0, "device": device,
          "uuid": str(getattr(props, "uuid", "")), "pci_bus_id": getattr(props, "pci_bus_id", None),
          "name": props.name, "exchange": exchange, "numa_cpus": numa}
    if world <= 1:
        return [me]
    out = [None] * world
    dist.all_gather_object(out, me, group=group)
    return out


def ring_spill(session, world: int, group=None) -> int:
    """Peer-HBM offload target for data-parallel runs: every rank hosts a
    spill buffer (its own plan's offload bytes; the plans are identical) and
    offloads into the buffer of rank (r + 1) % world, so offload/prefetch
    copies travel over NVLink to a neighbour's spare HBM instead of PCIe.
    The session must be created with offload_target="device". Returns the
    neighbour rank."""
    import torch.distributed as dist
    if world < 2:
        raise ValueError("a peer offload target needs at least two ranks")
    h = session.spill_export()
    handles = [None] * world
    dist.all_gather_object(handles, h, group=group)
    rank = dist.get_rank(group)
    peer = (rank + 1) % world
    session.spill_attach(handles[peer])
    return peer


class PeerUnavailable(RuntimeError):
    """Some rank could not map its peers' arenas (raised on every rank)."""


class PeerDataParallel:
    """Fused peer-memory gradient exchange + SGD (vdnn_session_peer_*). Wraps a
    Session created with external_grads=True; every rank of the process group
    must construct it (the IPC handles are all-gathered over ``group``)."""

    mode = "peer"

    def __init__(self, session, world: int, group=None, overlap: Optional[bool] = None):
        import torch.distributed as dist
        self.s = session
        self.world = world
        h = session.peer_export()
        if world > 1:
            handles = [None] * world
            dist.all_gather_object(handles, h, group=group)
            rank = dist.get_rank(group)
        else:
            handles, rank = [h], 0
        err = None
        try:
            session.peer_attach(rank, handles)
        except Exception as e:  # e.g. cudaIpcOpenMemHandle refused (no P2P path)
            err = repr(e)
        errs = [err]
        if world > 1:  # all ranks attach or none does: a lone attached rank would wait in the barrier
            errs = [None] * world
            dist.all_gather_object(errs, err, group=group)
        bad = [f"rank {r}: {e}" for r, e in enumerate(errs) if e]
        if bad:
            session.peer_detach()
            raise PeerUnavailable("; ".join(bad))
        if overlap is None:
            overlap = os.environ.get("VDNN_DP_OVERLAP", "1") != "0"
        self.overlap = bool(overlap)
        if self.overlap:
            session.peer_overlap(True, 1.0 / world)
            self.mode = "peer-overlap"

    def step(self, lr: float, want_loss: bool = False) -> Optional[float]:
        loss = self.s.step(lr, want_loss=want_loss)
        if not self.overlap:
            # after the step's kernels (the loss read inside step() happens
            # before the exchange completes)
            self.s.peer_exchange(lr, 1.0 / self.world)
        return loss

    def close(self) -> None:
        self.s.peer_detach()


class DataParallel:
    """NCCL all-reduce of the gradient arena, then SGD. Wraps a Session
    created with external_grads=True."""

    mode = "nccl"

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
