import sys, torch
sys.path.insert(0, "/root/repo")
from paper_2602_07263_b200.layer import FusedLoRALayer
from paper_2602_07263_b200.workload import config
wl = config("C2")
for proj in ("q", "gate", "down"):
    name, d, k = [p for p in wl.projections if p[0] == proj][0]
    g = torch.Generator(device="cuda").manual_seed(0)
    lay = FusedLoRALayer(d, k, wl.ranks)
    lay.set_base((torch.randn(d, k, generator=g, device="cuda") * d ** -0.5).bfloat16())
    for s, r in enumerate(wl.ranks):
        lay.set_adapter(s, (torch.randn(d, r, generator=g, device="cuda") * d ** -0.5).bfloat16(),
                        (torch.randn(r, k, generator=g, device="cuda") * r ** -0.5).bfloat16())
    T = wl.tokens
    X = torch.randn(T, d, generator=g, device="cuda").bfloat16()
    dY = torch.randn(T, k, generator=g, device="cuda").bfloat16()
    plan = lay.plan(wl.token_slots())
    H = torch.zeros(T, lay.R, dtype=torch.bfloat16, device="cuda"); dH = torch.zeros_like(H)
    dX = torch.empty(T, d, dtype=torch.bfloat16, device="cuda")
    lay.shrink(plan, X, H); lay.dh(plan, dY, dH)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    rd = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    def t(pre, n=20):
        ts = []
        for _ in range(n):
            pre()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); lay.grads(plan, H, dY, X, dH); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort(); return ts[len(ts) // 2]
    r = {"after_dX": t(lambda: lay.dx(plan, dY, dH, dX)),
         "after_write_flush": t(lambda: flush.zero_()),
         "after_read_flush": t(lambda: rd.sum()),
         "warm": t(lambda: None)}
    print(proj, {k: round(v, 1) for k, v in r.items()}, flush=True)
    lay.close()
