#!/usr/bin/env python
"""Headline benchmark: VGG-16 batch 256 training images/sec and peak GPU
memory under a 12 GiB HBM budget with vDNN_dyn, next to vDNN_all, vDNN_conv
and the no-offload baseline (BASELINE.json metric/config 4).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

One step = one full training iteration (forward, backward, SGD) of VGG-16 at
batch 256 per GPU on synthetic data (U[-1,1) NHWC images, uniform labels,
He-normal weights), replaying the bit-exact vDNN plan on the B200: offload and
prefetch copies over PCIe, all compute in sm_100a tcgen05 kernels. Inputs are
far larger than L2 (activations are GBs), so no explicit L2 flush is needed.
N > 1: data parallel, one process per GPU, per-rank batch 256 (weak scaling);
every step the weight gradients are exchanged by the fused peer-memory
reduce + SGD + broadcast kernel (VDNN_DP=nccl: NCCL all-reduce + SGD
instead); time = max over ranks.

--impl reference times the reference's CPU path on this host: the compiled
reference simulator's planning (dynamic_select + simulate, oracle/_ref) plus
the CPU numeric training step restated in oracle/numeric.py (torch CPU fp32,
all host threads) on a bounded sample batch.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

GIB12 = 12884901888
METRIC = "VGG-16 b256 train images/sec & peak GPU mem (vDNN_all/conv/dyn vs no-offload)"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


TRAFFIC_FILES = ("r02_conv_traffic.json", "r01_conv_traffic.json")  # newest capture first


def conv_traffic(key="conv_dram_bytes_per_launch"):
    """(mean DRAM bytes per launch, source file) from the newest committed ncu
    capture (profiles/r0N_conv_traffic.json; `key`: the whole conv engine or
    the dominant kernel), or (None, None)."""
    for name in TRAFFIC_FILES:
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", name)
        try:
            with open(path) as f:
                return int(json.load(f)[key]), "profiles/" + name
        except (OSError, KeyError, ValueError):
            continue
    return None, None


def pair_fprop_layers(g, es):
    """Conv layers whose FPROP runs the dominant kernel of the step -- the
    CTA-pair kernel (fp32 storage: tc_conv_pair_kernel, conv.cu launch():
    >= 256 output columns in 128-multiples and >= 148 pair tiles of 256 x 256;
    BF16: tcb_pair_kernel, >= 256 columns)."""
    import paper_1602_08124_b200 as V
    out = []
    for l in g.layers():
        if l.kind != V.LayerKind.Conv:
            continue
        sh = g.shape(l.id)
        co, m = sh.c, sh.n * sh.h * sh.w
        if es == 4 and co >= 256 and co % 128 == 0 and ((m + 255) // 256) * (co // 256) >= 148:
            out.append(l.id)
        elif es == 2 and co >= 256:
            out.append(l.id)
    return out


def measured_tf32_peak(peaks, peaks_src):
    """The TF32 roofline denominator: the tcgen05 kind::tf32 issue ceiling
    measured on this device (vdnn_kernel_tf32_peak: M128 N256 K8 MMAs back to
    back on every SM, no memory traffic). MEASURED_PEAKS.json has no TF32
    entry; its bf16 figure / 2 is the fallback if the probe fails."""
    import ctypes as C
    from paper_1602_08124_b200 import _lib as L
    best = 0.0
    for _ in range(5):  # best of 5 (the first runs can see a cold power/clock state)
        v = C.c_double(0.0)
        if L.lib().vdnn_kernel_tf32_peak(C.byref(v)) == 0:
            best = max(best, v.value)
    if best > 0:
        return best, ("measured live (best of 5): tcgen05.mma kind::tf32 M128xN256xK8 issue ceiling, "
                      "148 SMs (vdnn_kernel_tf32_peak)")
    return float(peaks.get("bf16_tflops_sustained", 1400.0)) / 2.0, f"fallback: {peaks_src} bf16 sustained / 2"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return PEAKS_FALLBACK, "fallback"


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.FIELDS,
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# --------------------------------------------------------------- helpers ----
def gemm_flops(g):
    """Algorithmic GEMM FLOPs of one iteration: conv fprop +
    wgrad + dgrad (no dgrad when the input is the raw INPUT), FC 3x fprop."""
    import paper_1602_08124_b200 as V
    cm = V.CostModel()
    total = 0.0
    for l in g.layers():
        if l.kind not in (V.LayerKind.Conv, V.LayerKind.Fc):
            continue
        f = cm.flops(g, l.id, False)
        raw = all(g.layer(q).kind == V.LayerKind.Input for q in l.inputs)
        total += f * (2 if raw else 3)
    return total


def memory_bound_bytes(g):
    """Algorithmic bytes of the memory-bound kernels per iteration:
    ReLU 2Y fwd + 3Y bwd; pool (X+Y) fwd + (2X+2Y) bwd; SGD 12 B/param."""
    import paper_1602_08124_b200 as V
    cm = V.CostModel()
    b = 0
    for l in g.layers():
        if l.kind == V.LayerKind.Actv:
            y = cm.tensor_bytes_of(g.shape(l.id))
            b += 5 * y
        elif l.kind == V.LayerKind.Pool:
            y = cm.tensor_bytes_of(g.shape(l.id))
            x = sum(cm.tensor_bytes_of(g.shape(q)) for q in l.inputs)
            b += 3 * (x + y)
        b += 3 * cm.weight_bytes(g, l.id)
    return b


def link_bandwidth(device: int, nbytes: int = 1 << 30):
    """Pinned cudaMemcpyAsync GB/s per direction (host-link roofline)."""
    import torch
    h = torch.empty(nbytes // 4, dtype=torch.float32, pin_memory=True)
    d = torch.empty(nbytes // 4, dtype=torch.float32, device=f"cuda:{device}")
    out = {}
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        best = 0.0
        for _ in range(3):
            s = torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event(enable_timing=True)
            s.record()
            fn()
            e.record()
            e.synchronize()
            best = max(best, nbytes / (s.elapsed_time(e) * 1e-3) / 1e9)
        out[name + "_gbs"] = round(best, 2)
    del h, d
    torch.cuda.empty_cache()  # give the probe's 1 GiB back before the sessions measure device usage
    return out


# ---------------------------------------------------------------- our arm ----
def run_policy(policy, args, device, world, peaks, want_e2e, sampler_cls):
    import numpy as np
    import torch
    import paper_1602_08124_b200 as V
    from paper_1602_08124_b200.dist import make_data_parallel, max_over_ranks

    g = V.build_preset(args.net, args.batch) if args.extra == 0 else V.extend_vgg(args.extra, args.batch)
    cm = V.CostModel()
    cap = args.capacity
    # "<policy>b": BF16 storage -- the reference's elem_size = 2
    # (cost_model.hpp:69): the planner sizes every tensor at 2 bytes (its own
    # decisions and schedule), the executor stores bf16 and runs kind::f16
    name = policy
    bf16 = policy.endswith("b")
    if bf16:
        policy = policy[:-1]
        cm.elem_size = 2
    # "<policy>z": the same plan with zero-value-compressed offload/prefetch;
    # "<policy>p": the same plan offloading into the ring neighbour's spare
    # HBM over NVLink (data parallel only: a peer GPU is the offload target)
    # "<policy>t": compressed, and maps read in backward only by TF32
    # contractions / ReLU masks travel TF32-exact (bit-identical step)
    # "<policy>f": fp32-accurate contractions (3xTF32) instead of TF32
    precise = args.precise or policy.endswith("f")
    if policy.endswith("f"):
        policy = policy[:-1]
    compress = "tf32" if policy.endswith("t") else policy.endswith("z")
    peer_target = policy.endswith("p")
    if compress or peer_target:
        policy = policy[:-1]
    if peer_target and world < 2:
        return {"policy": policy + "p", "verdict": "skipped: a peer-HBM offload target needs >= 2 GPUs"}
    sel = None
    if policy == "dyn":
        sel = V.dynamic_select(g, cap, cm)
        if sel.decision is None:
            return {"policy": policy, "verdict": "untrainable"}
        d = sel.decision
    elif policy == "all":
        d = V.static_decision(V.PolicyKind.VdnnAll, V.AlgoMode.MemoryOptimal, g, cm)
    elif policy == "conv":
        d = V.static_decision(V.PolicyKind.VdnnConv, V.AlgoMode.MemoryOptimal, g, cm)
    else:  # no-offload baseline(p) with the device's capacity as the budget
        d = V.static_decision(V.PolicyKind.Baseline, V.AlgoMode.PerfOptimal, g, cm)
        free, total = torch.cuda.mem_get_info(device)
        cap = int(free - (6 << 30))
        if world > 1:  # one plan on every rank (the peer exchange maps weights by offset)
            t = torch.tensor([cap], dtype=torch.int64,
                             device="cpu" if torch.distributed.get_backend() == "gloo" else f"cuda:{device}")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MIN)
            cap = int(t.item())
    free0, total0 = torch.cuda.mem_get_info(device)  # before the session: context + this process's torch state
    plan = V.simulate(g, d, cm, cap)
    if not plan.pass_:
        return {"policy": policy, "label": d.label, "verdict": plan.verdict(), "capacity": cap}
    s = V.Session(g, d, cm, cap, device=device, record_timeline=True, external_grads=world > 1,
                  precise_fp32=precise, compress_offload=compress,
                  offload_target="device" if peer_target else "host")
    if peer_target:
        from paper_1602_08124_b200.dist import ring_spill
        ring_spill(s, world)
    dp = make_data_parallel(s, world, device) if world > 1 else None

    def one(want_loss=False):
        return dp.step(args.lr, want_loss) if dp else s.step(args.lr, want_loss=want_loss)

    stream = torch.cuda.ExternalStream(s.stream, device=f"cuda:{device}")
    s.synthetic_batch(1234 + device)
    for _ in range(args.warmup):
        one()
    s.synchronize()
    torch.cuda.synchronize(device)
    if world > 1:
        torch.distributed.barrier()
    ts0 = s.transfer_stats()
    l0 = V.kernel_launch_count()
    s.pause_timeline(True)  # no per-op timing events inside the timed region (one more step records them below)
    with sampler_cls(device) as clk:
        # one event per step boundary on the session's compute stream: the
        # region [first, last] is the timed total, the gaps give the median
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
        evs[0].record(stream)
        for i in range(args.steps):
            one()
            evs[i + 1].record(stream)
        evs[-1].synchronize()
        ev0, ev1 = evs[0], evs[-1]
        per_step = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
    launches = V.kernel_launch_count() - l0
    ts1 = s.transfer_stats()
    wire = {k: (ts1[k] - ts0[k]) // args.steps for k in ts0}
    ms = ev0.elapsed_time(ev1) / args.steps
    ms = max_over_ranks(ms, world, device=f"cuda:{device}")
    imgs = args.batch * world / (ms * 1e-3)
    ms_median = max_over_ranks(statistics.median(per_step), world, device=f"cuda:{device}")
    s.pause_timeline(False)
    loss = s.step(args.lr, want_loss=True) if not dp else dp.step(args.lr, True)

    # per-layer measured times of that last step
    fwd_ms, bwd_ms = s.layer_times()
    m = s.measured_report()
    conv_ms = sum(fwd_ms[l.id] + bwd_ms[l.id] for l in g.layers() if l.kind in (V.LayerKind.Conv, V.LayerKind.Fc))
    kernel_ms = sum(fwd_ms) + sum(bwd_ms)
    mem_ms = sum(fwd_ms[l.id] + bwd_ms[l.id] for l in g.layers()
                 if l.kind in (V.LayerKind.Actv, V.LayerKind.Pool))
    flops = gemm_flops(g)
    conv_tflops = flops / (conv_ms * 1e-3) / 1e12 if conv_ms > 0 else None
    off_ms = sum((e.end - e.start) for e in m.events if e.kind == V.EventKind.Offload) * 1e-6
    pre_ms = sum((e.end - e.start) for e in m.events if e.kind == V.EventKind.Prefetch) * 1e-6
    free, total = torch.cuda.mem_get_info(device)
    if getattr(args, "artifacts", None) and name in ("dyn", "dynb") and device == 0:
        write_step_artifacts(args, name, g, d, cm, cap, s, m, sel)
    res = {
        "policy": name,
        "label": d.label + ({"tf32": " +zvc/tf32-exact", True: " +zvc"}.get(compress, ""))
                 + (" ->peer HBM" if peer_target else ""),
        "verdict": "PASS", "capacity_bytes": cap,
        "images_per_s": round(imgs, 2), "ms_per_step": round(ms, 3), "ms_per_step_median": round(ms_median, 3),
        "loss": loss, "precise_fp32": bool(precise), "storage": "bf16" if bf16 else "fp32",
        "peak_pool_bytes": plan.max_mem_bytes, "arena_bytes": s.arena_info()["arena_bytes"],
        "device_used_bytes": total - free,
        # process HBM = pool arena (<= the budget) + non-pool scratch + what was
        # in use before the session (CUDA context, torch)
        "hbm": {"arena_bytes": s.arena_info()["arena_bytes"], "non_pool_scratch_bytes": s.arena_info()["scratch_bytes"],
                "context_and_other_bytes": total0 - free0,
                "unaccounted_bytes": (total - free) - (total0 - free0) - s.arena_info()["arena_bytes"]
                                     - s.arena_info()["scratch_bytes"]},
        "offload_bytes_per_iter": plan.offload_traffic_bytes, "prefetch_bytes_per_iter": plan.prefetch_traffic_bytes,
        "d2h_gbs": round(plan.offload_traffic_bytes / (off_ms * 1e-3) / 1e9, 2) if off_ms > 0 else None,
        "h2d_gbs": round(plan.prefetch_traffic_bytes / (pre_ms * 1e-3) / 1e9, 2) if pre_ms > 0 else None,
        # exposed (non-overlapped) transfer time = the SYNC stalls of the
        # measured event log of one recorded step (simulator.hpp:315-322
        # forward: FWD(n+1) waits for n's offloads; :400-441 backward: BWD(m)
        # waits for its prefetches / the step's prefetch tail), re-timed from
        # CUDA events on both streams
        "exposed_transfer_ms": (round(m.stall_ns() * 1e-6, 3) if plan.offload_traffic_bytes > 0 else None),
        "stall_fwd_offload_ms": round(m.stall_fwd_offload_ns * 1e-6, 3),
        "stall_bwd_prefetch_ms": round(m.stall_bwd_prefetch_ns * 1e-6, 3),
        "measured_step_ms": round(m.total_ns * 1e-6, 3),
        "kernel_ms": round(kernel_ms, 3),
        "conv_fc_ms": round(conv_ms, 3), "memory_bound_ms": round(mem_ms, 3),
        "conv_fc_tflops": round(conv_tflops, 1) if conv_tflops else None,
        "gpu_launches": launches, "clocks": clk.summary(),
        "transfer": ("zero-value-compressed via SMs (zero-copy)" if compress else
                     "cudaMemcpyAsync to the ring neighbour's HBM (NVLink peer copies)" if peer_target else
                     "cudaMemcpyAsync (copy engines)"),
        "offload_wire_bytes_per_iter": wire["offload_wire"], "prefetch_wire_bytes_per_iter": wire["prefetch_wire"],
        "wire_ratio": round((wire["offload_wire"] + wire["prefetch_wire"]) /
                            max(1, wire["offload_planned"] + wire["prefetch_planned"]), 4),
        "signature": plan.signature(),
        "dp_exchange": (dp.mode if dp else None),
    }
    if want_e2e:
        # end to end through the public API: pinned host batch -> device every
        # step, loss read back every step
        sh = g.shape(0)
        rng = np.random.default_rng(99 + device)
        host_imgs = rng.uniform(-1, 1, size=(sh.n, sh.h, sh.w, sh.c)).astype(np.float32)
        if bf16:  # the loader hands the session its storage format
            host_imgs = V.to_bf16_bits(host_imgs).view(np.int16)
        imgs_h = torch.from_numpy(host_imgs).pin_memory()
        ls = g.shape(g.layer(g.size() - 1).inputs[0])
        labs_h = torch.from_numpy(rng.integers(0, ls.c, size=sh.n).astype(np.int32)).pin_memory()
        # input pipeline: each step's batch is staged (pinned host -> device)
        # on the session's input stream while the previous step runs; the
        # step moves it into the INPUT extent; every step's loss is read back,
        # pipelined one step behind (queue now, wait after the next step was
        # enqueued) so the host never idles the GPU
        pending = []

        def e2e_step():
            one(False)
            pending.append(s.queue_loss())
            s.prefetch_batch_ptr(imgs_h.data_ptr(), labs_h.data_ptr())
            if len(pending) > 1:
                s.wait_loss(pending.pop(0))

        s.pause_timeline(True)
        s.prefetch_batch_ptr(imgs_h.data_ptr(), labs_h.data_ptr())
        for _ in range(2):
            e2e_step()
        s.wait_loss(pending.pop(0))
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            e2e_step()
        s.wait_loss(pending.pop(0))  # the last step's loss is read back inside the timed region
        e1.record(stream)
        e1.synchronize()
        wall = (time.perf_counter() - t0) / args.steps
        ems = max(e0.elapsed_time(e1) / args.steps, wall * 1e3)
        ems = max_over_ranks(ems, world, device=f"cuda:{device}")
        res["e2e"] = {"value": round(args.batch * world / (ems * 1e-3), 2), "unit": "images/s",
                      "h2d_bytes_per_step": imgs_h.numel() * imgs_h.element_size() + labs_h.numel() * 4,
                      "d2h_bytes_per_step": 4,
                      "ms_per_step": round(ems, 3)}
    res["_flops"] = flops
    res["_conv_ms"] = conv_ms
    # the dominant kernel's FPROP launches of the measured step (per-op CUDA
    # events on the compute stream): algorithmic FLOPs per launch and time
    dom = pair_fprop_layers(g, cm.elem_size)
    res["_dom_n"] = len(dom)
    res["_dom_flops"] = sum(cm.flops(g, i, False) for i in dom)
    res["_dom_ms"] = sum(fwd_ms[i] for i in dom)
    del s
    torch.cuda.synchronize(device)
    return res


def write_step_artifacts(args, name, g, d, cm, cap, s, m, sel):
    """--artifacts DIR: the reference's artefact files (report.hpp:44-236) for
    the measured step, plus the calibrated re-plan: every
    layer's latency pinned to its measured time, the link to its measured
    bandwidth; the schedule must not move, the planned time should track the
    measured one."""
    import paper_1602_08124_b200 as V
    from paper_1602_08124_b200 import formats as F
    out = os.path.join(args.artifacts, f"{args.net}{'' if args.extra == 0 else '+' + str(args.extra)}_b{args.batch}_{name}")
    F.write_artifacts(out, g, d, m, sel.passes if sel else None)
    xfer = [e for e in m.events if e.kind in (V.EventKind.Offload, V.EventKind.Prefetch)]
    ns = sum(e.end - e.start for e in xfer)
    gbs = sum(e.bytes for e in xfer) / ns if ns else None
    cal = F.calibrated_cost_model(s, link_gbs=gbs)
    r = V.simulate(g, d, cal, cap)
    summary = {
        "decision": d.label, "elem_size": cm.elem_size, "capacity": cap,
        "measured_step_ns": m.total_ns, "measured_stall_ns": m.stall_ns(),
        "default_model_plan_ns": s.plan.total_ns,
        "calibrated_plan_ns": r.total_ns, "calibrated_stall_ns": r.stall_ns(),
        "calibrated_rel_err": (r.total_ns - m.total_ns) / m.total_ns,
        "link_gbs_measured": gbs,
        "signature_planned": s.plan.signature(), "signature_calibrated": r.signature(),
        "replay_violations": [v.kind for v in V.replay_check(m, g, d, cap)],
    }
    with open(os.path.join(out, "calibration.json"), "w") as f:
        json.dump(summary, f, indent=1)


_CPU_WARM = False


def cpu_baseline_sample(args, seconds_target=15.0):
    """Reference CPU path on this host: the compiled reference planner
    (dynamic_select + simulate, oracle/_ref) + the numeric restatement of one
    training iteration (torch CPU fp32, all threads) on a small batch. The
    graphs come from the reference's own presets (refsim.preset_spec) so this
    arm never loads the product library (libvdnn.so)."""
    import numpy as np
    import torch
    from oracle import numeric, refsim
    cores = os.cpu_count() or 1
    torch.set_num_threads(cores)
    sample_batch = args.cpu_sample_batch
    g = numeric.layers_of(refsim.preset_spec(args.net, sample_batch, args.extra))
    full_spec = refsim.preset_spec(args.net, args.batch, args.extra)
    plan_s = refsim.time_plan(full_spec, args.capacity, 20)
    w = numeric.he_weights(g)
    sh = g[0].shape  # NCHW
    rng = np.random.default_rng(5)
    images = rng.uniform(-1, 1, size=(sh[0], sh[2], sh[3], sh[1])).astype(np.float32)
    classes = int(np.prod(g[g[-1].inputs[0]].shape[1:]))
    labels = rng.integers(0, classes, size=sh[0]).astype(np.int32)
    global _CPU_WARM
    if not _CPU_WARM:  # first call: torch CPU thread pool / allocator warm-up on a tiny batch, untimed
        gw = numeric.layers_of(refsim.preset_spec(args.net, 2, args.extra))
        shw = gw[0].shape
        numeric.train_step(gw, numeric.he_weights(gw),
                           rng.uniform(-1, 1, size=(shw[0], shw[2], shw[3], shw[1])).astype(np.float32),
                           rng.integers(0, classes, size=shw[0]).astype(np.int32), args.lr, dtype=torch.float32)
        _CPU_WARM = True
    t0 = time.perf_counter()
    numeric.train_step(g, w, images, labels, args.lr, dtype=torch.float32)
    step_s = time.perf_counter() - t0
    return {"value": round(sample_batch / (step_s + plan_s), 3), "unit": "images/s", "cores": cores,
            "kind": "port",
            "sample": (f"{args.net} batch {sample_batch}: reference planner (oracle/_ref dynamic_select+simulate "
                       f"at b{args.batch}, {plan_s * 1e3:.2f} ms) + CPU numeric fwd/bwd/SGD step "
                       f"(oracle/numeric.py, torch fp32, {cores} threads, {step_s:.2f} s)")}, step_s + plan_s


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    steps = []
    for i in range(args.warmup + args.steps):
        base, secs = cpu_baseline_sample(args)
        if i >= args.warmup:
            steps.append(secs)
    ms = statistics.mean(steps) * 1e3
    value = args.cpu_sample_batch / (ms * 1e-3)
    base["value"] = round(value, 3)
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "images/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 2),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{args.net} batch {args.batch} vDNN_dyn @ {args.capacity} B (CPU sample batch "
                                   f"{args.cpu_sample_batch})", "global_batch": args.cpu_sample_batch},
            "cpu_baseline": base,
            "e2e": {"value": round(value, 3), "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--net", default="vgg16")
    ap.add_argument("--extra", type=int, default=0, help="extend_vgg extra conv layers (400 -> VGG-416)")
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--capacity", type=int, default=GIB12)
    ap.add_argument("--policies", default=None,
                    help="dyn/all/conv/none; a trailing z = same plan with compressed offload, t = compressed with "
                         "TF32-exact values where only TF32 contractions read the map, a trailing p = "
                         "offload into a peer GPU's HBM (N > 1), a trailing f = fp32-accurate 3xTF32 "
                         "contractions, a trailing b = BF16 storage (elem_size 2: its own plan). Default: "
                         "dyn,dynz,dynt,all,conv,none,dynf,nonef,dynb,dynzb,noneb (N > 1: dyn,dynp,dynz,dynt,all,conv,none)")
    ap.add_argument("--lr", type=float, default=0.01)
    ap.add_argument("--precise", action="store_true", help="3xTF32 fp32-accurate contractions")
    ap.add_argument("--cpu-sample-batch", type=int, default=96,
                    help="images in the CPU reference sample (~7 s of CPU work for VGG-16 b96 on 16 cores)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--artifacts", default=None,
                    help="write report.json / timeline.csv / pool_trace.csv / decision.json / graph.json / "
                         "profile_passes.csv / calibration.json of the measured dyn (and dynb) step into DIR")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    from paper_1602_08124_b200.dist import env_rank
    rank, local, world = env_rank()
    if world > 1:
        if os.environ.get("VDNN_BENCH_SAME_DEVICE") == "1":
            # test hook: every rank on cuda:0 (the one-GPU box), gloo for the
            # host collectives; the peer exchange still runs over CUDA IPC
            local = 0
            torch.cuda.set_device(0)
            torch.distributed.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            os.environ.setdefault("NCCL_DEBUG", "INFO")  # the NCCL rank census (NVLS / P2P paths) in stderr
            torch.distributed.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    device = local
    torch.cuda.set_device(device)
    from paper_1602_08124_b200.dist import bind_numa, rank_census
    numa = bind_numa(device)  # before any pinned host arena is allocated
    peaks, peaks_src = load_peaks()
    link = link_bandwidth(device)
    # the TF32 ceiling is probed first, on a cool GPU at full clocks: the dyn
    # step's conv kernels run at those clocks (the link-bound step leaves the
    # GPU mostly idle), while a probe after the no-offload run measured the
    # power-capped clock (835 vs 1,095 TFLOP/s)
    tf32_peak, peak_note = measured_tf32_peak(peaks, peaks_src)

    if args.policies is None:
        args.policies = ("dyn,dynz,dynt,all,conv,none,dynf,nonef,dynb,dynzb,noneb" if world == 1
                         else "dyn,dynp,dynz,dynt,all,conv,none")
    results = {}
    for p in [x for x in args.policies.split(",") if x]:
        results[p] = run_policy(p, args, device, world, peaks, want_e2e=(p in ("dyn", "dynb")),
                                sampler_cls=ClockSampler)

    head = results.get("dyn") or next(iter(results.values()))
    census = rank_census(world, device, head.get("dp_exchange"), numa) if world > 1 else None
    line = {
        "metric": METRIC, "value": head.get("images_per_s"), "unit": "images/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": head.get("ms_per_step"),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 (tf32 tensor cores)" if not args.precise else "f32 (3xtf32)",
        "data": "synthetic (U[-1,1) NHWC images, uniform labels, He-normal init)",
        "config": {"workload": f"{args.net}{'' if args.extra == 0 else '+' + str(args.extra)} batch {args.batch}/GPU, "
                               f"vDNN_dyn under {args.capacity} B HBM budget ({head.get('label')})",
                   "global_batch": args.batch * world, "per_gpu_batch": args.batch,
                   "capacity_bytes": args.capacity, "parallelism": f"dp{world}",
                   "gradient_exchange": (None if world == 1 else head.get("dp_exchange")),
                   "l2": "inputs larger than L2 (activation maps are GBs); no flush needed"},
        "e2e": head.get("e2e"),
        "gpu_launches": head.get("gpu_launches"),
        "clocks": head.get("clocks"),
        "peak_gpu_mem_bytes": head.get("peak_pool_bytes"),
        "device_used_bytes": head.get("device_used_bytes"),
        "hbm": head.get("hbm"),
    }
    if census:
        line["rank_census"] = census
    if head.get("_conv_ms"):
        ach = head["_flops"] / (head["_conv_ms"] * 1e-3) / 1e12
        engine = {"kernels": "every conv+FC fprop, dgrad, wgrad launch of the step (tc_conv_pair / tc_wgrad_pair / "
                             "tc_conv_halo_pair / tc_wgrad_halo_pair / tc_conv / tc_conv_persist / c3tc)",
                  "achieved": round(ach, 1), "frac": round(ach / tf32_peak, 4),
                  "traffic": conv_traffic()[0],
                  "traffic_note": f"mean DRAM read+write bytes per conv-engine launch, ncu {conv_traffic()[1]}"}
        bf = (peaks or {}).get("bf16_tflops")
        if head.get("_dom_ms"):
            # the dominant kernel (39% of the dyn step's serialized kernel time,
            # profiles/r02s4_launches_vgg16_b256_dyn_summary.txt): its FPROP
            # launches, algorithmic FLOPs (2 k^2 Cin Cout Ho Wo N each) over
            # their CUDA-event durations in the measured step
            dach = head["_dom_flops"] / (head["_dom_ms"] * 1e-3) / 1e12
            line["roofline"] = {
                "bound": "tensor",
                "kernel": f"tc_conv_pair_kernel<5,1,4> (TF32 CTA pair, M256xN256xK8): the FPROP launches of the "
                          f"{head['_dom_n']} conv layers with >= 256 output channels",
                "achieved": round(dach, 1), "peak": round(tf32_peak, 1), "unit": "TFLOP/s",
                "frac": round(dach / tf32_peak, 4),
                "frac_of_half_bf16_burst": (round(dach / (bf / 2), 4) if bf else None),
                "traffic": conv_traffic("pair_dram_bytes_per_launch")[0],
                "peak_note": peak_note + ("; kind::tf32 runs at half the f16 rate, so MEASURED_PEAKS' bf16 burst "
                                          f"{bf} TFLOP/s / 2 is the other denominator" if bf else ""),
                "traffic_note": "mean DRAM read+write bytes per tc_conv_pair_kernel launch of one dyn step, ncu "
                                f"{conv_traffic('pair_dram_bytes_per_launch')[1]}",
                "engine": engine}
        else:
            line["roofline"] = dict({"bound": "tensor", "kernel": "tcgen05 conv engine", "achieved": engine["achieved"],
                                     "peak": round(tf32_peak, 1), "unit": "TFLOP/s", "frac": engine["frac"],
                                     "traffic": engine["traffic"], "peak_note": peak_note}, engine=engine)
    line["host_link"] = dict(link, **{
        "offload_bytes_per_iter": head.get("offload_bytes_per_iter"),
        "d2h_gbs_in_run": head.get("d2h_gbs"), "h2d_gbs_in_run": head.get("h2d_gbs"),
        "exposed_transfer_ms": head.get("exposed_transfer_ms")})
    pol = {}
    for k, r in results.items():
        pol[k] = {kk: vv for kk, vv in r.items() if not kk.startswith("_") and kk not in ("clocks", "e2e")}
        if r.get("clocks"):
            pol[k]["sm_mhz_median"] = r["clocks"].get("sm_mhz")
    if "none" in results and results["none"].get("images_per_s") and head.get("images_per_s"):
        line["slowdown_vs_no_offload"] = round(results["none"]["ms_per_step"] and
                                               head["ms_per_step"] / results["none"]["ms_per_step"], 4)
    line["policies"] = pol
    if "dynz" in results and results["dynz"].get("images_per_s"):
        z = results["dynz"]
        line["compressed_offload"] = {
            "policy": "vDNN_dyn, same plan, zero-value-compressed offload/prefetch (lossless, bit-identical)",
            "images_per_s": z["images_per_s"], "ms_per_step": z["ms_per_step"], "wire_ratio": z.get("wire_ratio"),
            "speedup_vs_copy_engines": round(z["images_per_s"] / head["images_per_s"], 3)
            if head.get("images_per_s") else None}
    if "dynt" in results and results["dynt"].get("images_per_s"):
        z = results["dynt"]
        line["tf32_exact_offload"] = {
            "policy": "vDNN_dyn, same plan, compressed offload/prefetch; maps read in backward only by TF32 "
                      "contractions and ReLU masks travel TF32-exact (bit-identical training step)",
            "images_per_s": z["images_per_s"], "ms_per_step": z["ms_per_step"], "wire_ratio": z.get("wire_ratio"),
            "speedup_vs_copy_engines": round(z["images_per_s"] / head["images_per_s"], 3)
            if head.get("images_per_s") else None}
    if any(k in results for k in ("dynf", "nonef")):
        line["fp32_accurate"] = {
            "policy": "3xTF32 contractions (fp32-accurate), same plans",
            **{k: {"images_per_s": results[k].get("images_per_s"), "ms_per_step": results[k].get("ms_per_step")}
               for k in ("dynf", "nonef") if k in results}}
    if "dynb" in results and results["dynb"].get("images_per_s"):
        z = results["dynb"]
        bf = peaks.get("bf16_tflops")  # burst: the conv/FC launches are timed one by one
        line["bf16_storage"] = {
            "policy": "BF16 storage (the reference's elem_size = 2, cost_model.hpp:69): its own vDNN_dyn plan "
                      f"({z.get('label')}), kind::f16 tensor cores, fp32 accumulation",
            "images_per_s": z["images_per_s"], "ms_per_step": z["ms_per_step"],
            "e2e_images_per_s": (z.get("e2e") or {}).get("value"),
            "offload_bytes_per_iter": z.get("offload_bytes_per_iter"), "peak_pool_bytes": z.get("peak_pool_bytes"),
            "exposed_transfer_ms": z.get("exposed_transfer_ms"), "conv_fc_tflops": z.get("conv_fc_tflops"),
            "conv_fc_frac_of_bf16_peak": (round(z["conv_fc_tflops"] / bf, 4) if bf and z.get("conv_fc_tflops")
                                          else None),
            "no_offload_images_per_s": results.get("noneb", {}).get("images_per_s"),
            "slowdown_vs_bf16_no_offload": (round(z["ms_per_step"] / results["noneb"]["ms_per_step"], 4)
                                            if results.get("noneb", {}).get("ms_per_step") else None),
            "speedup_vs_fp32_dyn": (round(z["images_per_s"] / head["images_per_s"], 3)
                                    if head.get("images_per_s") else None)}
        zb = results.get("dynzb", {})
        if zb.get("images_per_s"):
            # the same BF16 plan with lossless zero-value-compressed transfers (bit-identical step)
            line["bf16_storage"]["compressed_offload"] = {
                "images_per_s": zb["images_per_s"], "ms_per_step": zb["ms_per_step"],
                "wire_ratio": zb.get("wire_ratio"), "exposed_transfer_ms": zb.get("exposed_transfer_ms"),
                "slowdown_vs_bf16_no_offload": (round(zb["ms_per_step"] / results["noneb"]["ms_per_step"], 4)
                                                if results.get("noneb", {}).get("ms_per_step") else None)}
    if "dynp" in results and results["dynp"].get("images_per_s"):
        z = results["dynp"]
        line["peer_hbm_offload"] = {
            "policy": "vDNN_dyn, same plan, offload target = ring neighbour's spare HBM (NVLink peer copies)",
            "images_per_s": z["images_per_s"], "ms_per_step": z["ms_per_step"],
            "offload_gbs": z.get("d2h_gbs"), "prefetch_gbs": z.get("h2d_gbs"),
            "slowdown_vs_no_offload": (round(z["ms_per_step"] / results["none"]["ms_per_step"], 4)
                                       if results.get("none", {}).get("ms_per_step") else None)}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        base, _ = cpu_baseline_sample(args)
        line["cpu_baseline"] = base
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
