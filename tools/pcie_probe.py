"""Raw pinned-host <-> device copy bandwidth (the e2e path's PCIe ceiling).

  python tools/pcie_probe.py
"""
import torch
for mb in (256, 1024):
    h = torch.empty(mb << 20, dtype=torch.uint8).pin_memory()
    d = torch.empty(mb << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): d.copy_(h, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    print(f"H2D {mb} MB: {10 * (mb << 20) / (e0.elapsed_time(e1) / 1e3) / 1e9:.1f} GB/s")
    e0.record()
    for _ in range(10): h.copy_(d, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    print(f"D2H {mb} MB: {10 * (mb << 20) / (e0.elapsed_time(e1) / 1e3) / 1e9:.1f} GB/s")

# several copy streams at once (the e2e path may split its inputs over copy engines)
for nstreams in (1, 2, 4):
    mb = 512
    hs = [torch.empty(mb << 20, dtype=torch.uint8).pin_memory() for _ in range(nstreams)]
    ds = [torch.empty(mb << 20, dtype=torch.uint8, device="cuda") for _ in range(nstreams)]
    ss = [torch.cuda.Stream() for _ in range(nstreams)]
    for _ in range(2):
        for h, d, s in zip(hs, ds, ss):
            with torch.cuda.stream(s):
                d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    e0.record(cur)
    for s in ss:
        s.wait_stream(cur)
    for _ in range(8):
        for h, d, s in zip(hs, ds, ss):
            with torch.cuda.stream(s):
                d.copy_(h, non_blocking=True)
    for s in ss:
        cur.wait_stream(s)
    e1.record(cur)
    torch.cuda.synchronize()
    tot = 8 * nstreams * (mb << 20)
    print(f"H2D {nstreams} streams x {mb} MB: {tot / (e0.elapsed_time(e1) / 1e3) / 1e9:.1f} GB/s")
