"""Development aid: pinned host <-> device copy rates on this box (the e2e bound of bench.py):
one 657 MB H2D copy (the per-step inputs) on 1 / 2 / 4 streams, and H2D concurrent with a D2H.
    python scripts/h2d_probe.py"""
import torch, time
dev = torch.device("cuda", 0)
n = 657113088 // 2
h = torch.empty(n, dtype=torch.bfloat16).pin_memory()
d = torch.empty(n, dtype=torch.bfloat16, device=dev)
h2 = [h[: n // 2], h[n // 2:]]
d2 = [d[: n // 2], d[n // 2:]]
streams = [torch.cuda.Stream() for _ in range(4)]
def one():
    d.copy_(h, non_blocking=True)
def two():
    for i in range(2):
        with torch.cuda.stream(streams[i]):
            d2[i].copy_(h2[i], non_blocking=True)
    for s in streams[:2]:
        torch.cuda.current_stream().wait_stream(s)
def four():
    parts = 4
    hs = h.chunk(parts); ds = d.chunk(parts)
    for i in range(parts):
        with torch.cuda.stream(streams[i]):
            ds[i].copy_(hs[i], non_blocking=True)
    for s in streams[:parts]:
        torch.cuda.current_stream().wait_stream(s)
hd = torch.empty(n // 3, dtype=torch.bfloat16).pin_memory()
dd = torch.empty(n // 3, dtype=torch.bfloat16, device=dev)
def duplex():
    with torch.cuda.stream(streams[0]):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(streams[1]):
        hd.copy_(dd, non_blocking=True)
    for s in streams[:2]:
        torch.cuda.current_stream().wait_stream(s)
for name, fn in (("1 stream", one), ("2 streams", two), ("4 streams", four), ("h2d 657MB + d2h 219MB concurrently", duplex)):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"{name}: {ms:.2f} ms, {657113088 / ms / 1e6:.1f} GB/s (h2d bytes)")
