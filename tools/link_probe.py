"""Host-link probe: pinned D2H / H2D GB/s with one copy stream vs the same
bytes split across two (or four) streams (copy engines), per direction and
bidirectional."""
import torch

GB = 1 << 30
n = 4 * GB // 4
dev = torch.empty(n, device="cuda")
host = torch.empty(n, pin_memory=True)
dev2 = torch.empty(n, device="cuda")
host2 = torch.empty(n, pin_memory=True)


def run(direction, nstreams, reps=3):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    chunk = n // nstreams
    best = 0.0
    for _ in range(reps):
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for i, st in enumerate(streams):
            st.wait_event(s)
            with torch.cuda.stream(st):
                sl = slice(i * chunk, (i + 1) * chunk)
                if direction in ("d2h", "both"):
                    host[sl].copy_(dev[sl], non_blocking=True)
                if direction in ("h2d", "both"):
                    dev2[sl].copy_(host2[sl], non_blocking=True)
        for st in streams:
            e.wait(st) if hasattr(e, "wait") else None
            torch.cuda.current_stream().wait_stream(st)
        e.record()
        e.synchronize()
        ms = s.elapsed_time(e)
        nbytes = 4 * n * (2 if direction == "both" else 1)
        best = max(best, nbytes / ms / 1e6)
    return best


for d in ("d2h", "h2d", "both"):
    print(d, {k: round(run(d, k), 2) for k in (1, 2, 4)}, "GB/s")
