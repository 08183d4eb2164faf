"""Step driver for the fused multi-LoRA layer set (the caller of the hot path).

One SSM layer-set step = forward of every adapted projection, then backward of every
projection in reverse order (synthetic upstream gradients dY), adapter gradients
accumulated in the layers' fp32 buffers. This is the per-iteration body of the
reference simulator's loop (proj/include/lora_fleet/sim_engine.hpp:306-315, paper
Alg. 1 FusedKernelLaunch) executed for real.
"""
from __future__ import annotations

import os

import torch

from .layer import FusedLoRALayer
from .workload import INPUT_GROUP, Workload


class LayerSetStep:
    """Forward/backward/optimizer driver for `wl.layers` stacked layer sets.

    Every (layer, projection) has its own frozen W, adapters, optimizer state and H stash
    (the backward of layer L consumes the H its forward produced). One tile plan per
    projection shape serves all layers (same registry layout). Activation buffers (X, Y,
    dY, dX) are shared across layers: the layer is the unit of work here and attention /
    norms / activations between projections are out of scope, so synthetic inputs stand in
    for them.
    """

    def __init__(self, wl: Workload, device: int = 0, seed: int | None = None,
                 shuffle: bool = False, y_dtype=torch.bfloat16, chain: bool = True,
                 keep_weights: bool = False):
        self.wl = wl
        # keep_weights: retain the bf16 W / A_j / B_j each layer was loaded with (the
        # full-size parity tests restate the step from them; the bench does not keep them)
        self.weights = {} if keep_weights else None
        # chain: each projection's shrink (forward) / dH (backward) rides as extra tiles in
        # the previous projection's fused GEMM launch (tlora_forward_gemm_shrink /
        # tlora_backward_dx_dh) instead of its own launch; bit-identical either way.
        self.chain = chain
        self.device = device
        dev = torch.device("cuda", device)
        self.dev = dev
        g = torch.Generator(device=dev)
        g.manual_seed(wl.seed if seed is None else seed)
        T = wl.tokens
        self.T = T
        self.slots = wl.token_slots(shuffle=shuffle)
        # interleaved tokens: gathered plans (job-sorted operands, one rank window per tile)
        # unless TLORA_GATHERED=0 (plain plans: wide K-extension windows, gathers per grads)
        import os
        self.gathered = bool(shuffle) and os.environ.get("TLORA_GATHERED", "1") != "0"
        self.layers, self.plans = {}, {}
        self.X, self.Y, self.H, self.dY, self.dX = {}, {}, {}, {}, {}
        self.keys = [(L, name) for L in range(wl.layers) for name, _, _ in wl.projections]
        dims = {name: (d, k) for name, d, k in wl.projections}
        for L, name in self.keys:
            d, k = dims[name]
            lay = FusedLoRALayer(d, k, wl.ranks, device=device)
            W = torch.randn(d, k, generator=g, device=dev, dtype=torch.float32).mul_(d ** -0.5)
            W = W.bfloat16()
            lay.set_base(W)
            ab = []
            for s, j in enumerate(wl.jobs):
                A = torch.randn(d, j.rank, generator=g, device=dev).mul_(d ** -0.5).bfloat16()
                B = torch.randn(j.rank, k, generator=g, device=dev).mul_(j.rank ** -0.5).bfloat16()
                lay.set_adapter(s, A, B)
                ab.append((A, B))
            if self.weights is not None:
                self.weights[(L, name)] = (W, ab)
            del W, ab
            self.layers[(L, name)] = lay
            if name not in self.plans:
                self.plans[name] = lay.plan(self.slots, gathered=self.gathered)
            grp = INPUT_GROUP.get(name, name)
            if grp not in self.X:
                self.X[grp] = torch.randn(T, d, generator=g, device=dev).bfloat16()
            if name not in self.Y:
                self.Y[name] = torch.empty(T, k, dtype=y_dtype, device=dev)
                self.dY[name] = torch.randn(T, k, generator=g, device=dev).bfloat16()
                self.dX[name] = torch.empty(T, d, dtype=torch.bfloat16, device=dev)
        if self.gathered:
            self.gX = {g: torch.empty_like(t) for g, t in self.X.items()}
            self.gdY = {n: torch.empty_like(t) for n, t in self.dY.items()}
        # H stashes: one zeroed arena; the masked low-rank launches only ever write each
        # token's window columns (zeros outside its own slot), so the rest stays zero
        R = self.layers[self.keys[0]].R  # packed rank width: same for every projection
        self.H_arena = torch.zeros(len(self.keys), T, R, dtype=torch.bfloat16, device=dev)
        for i, key in enumerate(self.keys):
            self.H[key] = self.H_arena[i]
        self.dH2 = torch.zeros(2, T, R, dtype=torch.bfloat16, device=dev)  # chained dH ping-pong
        torch.cuda.synchronize(dev)

    def x_of(self, name):
        X = self.gX if self.gathered else self.X
        return X[INPUT_GROUP.get(name, name)]

    def dy_of(self, name):
        return (self.gdY if self.gathered else self.dY)[name]

    def gather_inputs(self, stream=None):
        """Gathered plans: job-sorted copies of this step's inputs (X groups, dY), four
        tensors per launch; the fused GEMMs write Y / dX back in token order."""
        if not self.gathered:
            return
        pl = next(iter(self.plans.values()))
        pairs = [(self.X[g], self.gX[g]) for g in self.X] + \
                [(self.dY[n], self.gdY[n]) for n in self.dY]
        pl.gather(pairs, stream=stream)

    def forward(self, stream=None):
        self.gather_inputs(stream)
        if self.chain:
            import os
            return self.forward_chained(stream, os.environ.get("TLORA_PREFETCH_DH", "1") != "0")
        for L, name in self.keys:
            self.layers[(L, name)].forward(self.plans[name], self.x_of(name), self.Y[name],
                                           self.H[(L, name)], stream=stream)

    def _first_dh_buffer(self):
        return self.dH4[0] if getattr(self, "side_grads", False) else self.dH2[0]

    def forward_chained(self, stream=None, prefetch_dh: bool = True):
        """prefetch_dh: the last forward launch also computes the backward's first dH (the
        last projection's, from its upstream gradient dY) as extra tiles
        (tlora_forward_gemm_dh), so the backward starts with a fused dX launch."""
        keys = self.keys
        k0 = keys[0]
        self.layers[k0].shrink(self.plans[k0[1]], self.x_of(k0[1]), self.H[k0], stream=stream)
        for i, (L, name) in enumerate(keys):
            lay, pl = self.layers[(L, name)], self.plans[name]
            if i + 1 < len(keys):
                nk = keys[i + 1]
                lay.fused_gemm_shrink(pl, self.x_of(name), self.H[(L, name)], self.Y[name],
                                      self.layers[nk], self.plans[nk[1]], self.x_of(nk[1]),
                                      self.H[nk], zero_next=False, stream=stream)
            elif prefetch_dh:
                lay.fused_gemm_dh(pl, self.x_of(name), self.H[(L, name)], self.Y[name], lay, pl,
                                  self.dy_of(name), self._first_dh_buffer(), zero_next=False,
                                  stream=stream)
                self._dh_prefetched = True
            else:
                lay.fused_gemm(pl, self.x_of(name), self.H[(L, name)], self.Y[name], stream=stream)

    def enable_side_grads(self):
        """Chained backward with each projection's dB+dA launch on a side stream: it reads
        only H, X, dY and the projection's dH (produced by the previous dX launch), so it
        can run while the main stream's next fused GEMM runs, filling that GEMM's tail. dH
        uses a ring of buffers; a dX launch waits for the side-stream reader of the
        buffer it overwrites (ring depth TLORA_DH_RING, default 8: 0.7% faster than 4 on C2)."""
        self.side = torch.cuda.Stream(self.dev)
        self.dh_ring = max(2, int(os.environ.get("TLORA_DH_RING", "8")))
        self.dH4 = torch.zeros(self.dh_ring, self.T, self.dH2.shape[2], dtype=torch.bfloat16, device=self.dev)
        self.side_grads = True

    def _backward_side(self, main, beta, on_layer_done, opt_inline=False):
        side, keys = self.side, list(reversed(self.keys))
        ev = torch.cuda.Event()
        ev.record(main)
        side.wait_event(ev)  # adapters / grads of the previous step are settled
        done = {}            # key index -> event after its grads launch (side stream)
        k0 = keys[0]
        if not getattr(self, "_dh_prefetched", False):
            self.layers[k0].dh(self.plans[k0[1]], self.dy_of(k0[1]), self.dH4[0], stream=main)
        self._dh_prefetched = False
        for i, (L, name) in enumerate(keys):
            lay, pl = self.layers[(L, name)], self.plans[name]
            nr = self.dh_ring
            dH = self.dH4[i % nr]
            if i + 1 < len(keys):
                nk = keys[i + 1]
                if i + 1 - nr in done:  # buffer (i+1)%nr was last read by grads(i+1-nr)
                    main.wait_event(done[i + 1 - nr])
                lay.dx_dh(pl, self.dy_of(name), dH, self.dX[name], self.layers[nk], self.plans[nk[1]],
                          self.dy_of(nk[1]), self.dH4[(i + 1) % nr], zero_next=False, stream=main)
            else:
                lay.dx(pl, self.dy_of(name), dH, self.dX[name], stream=main)
            ready = torch.cuda.Event()
            ready.record(main)  # dH(i) was written by the previous launch on main
            side.wait_event(ready)
            lay.grads(pl, self.H[(L, name)], self.dy_of(name), self.x_of(name), dH, beta=beta,
                      stream=side)
            if opt_inline:  # nothing later in the step reads this projection's adapters
                lay.optimizer_step(stream=side)
            done[i] = torch.cuda.Event()
            done[i].record(side)
            if on_layer_done is not None:
                on_layer_done((L, name), lay, done[i])
        main.wait_stream(side)

    def backward_chained(self, stream=None, beta: float = 0.0, on_layer_done=None,
                         opt_inline=False):
        if getattr(self, "side_grads", False):
            return self._backward_side(stream if stream is not None else torch.cuda.current_stream(self.dev),
                                       beta, on_layer_done, opt_inline)
        keys = list(reversed(self.keys))
        k0 = keys[0]
        if not getattr(self, "_dh_prefetched", False):
            self.layers[k0].dh(self.plans[k0[1]], self.dy_of(k0[1]), self.dH2[0], stream=stream)
        self._dh_prefetched = False
        for i, (L, name) in enumerate(keys):
            lay, pl = self.layers[(L, name)], self.plans[name]
            dH = self.dH2[i % 2]
            if i + 1 < len(keys):
                nk = keys[i + 1]
                lay.dx_dh(pl, self.dy_of(name), dH, self.dX[name], self.layers[nk], self.plans[nk[1]],
                          self.dy_of(nk[1]), self.dH2[(i + 1) % 2], zero_next=False, stream=stream)
            else:
                lay.dx(pl, self.dy_of(name), dH, self.dX[name], stream=stream)
            lay.grads(pl, self.H[(L, name)], self.dy_of(name), self.x_of(name), dH, beta=beta,
                      stream=stream)
            if on_layer_done is not None:
                on_layer_done((L, name), lay)

    def backward(self, stream=None, beta: float = 0.0, on_layer_done=None):
        if self.chain:
            return self.backward_chained(stream, beta, on_layer_done)
        for L, name in reversed(self.keys):
            lay = self.layers[(L, name)]
            lay.backward(self.plans[name], self.dy_of(name), self.x_of(name), self.H[(L, name)],
                         self.dX[name], beta=beta, stream=stream)
            if on_layer_done is not None:
                on_layer_done((L, name), lay)

    # ---- overlapped schedule: low-rank launches on a side stream, fused GEMMs on the main
    def enable_overlap(self, lowrank_sms: int = -1):
        """Run the HBM-bound low-rank launches (shrink, dH, dA, dB) on a side stream with a
        small persistent grid, concurrently with the tensor-bound fused GEMMs (fwd, dX) on
        the main stream, which keep the remaining SMs (tlora_set_sm_budget)."""
        from . import capi
        total = torch.cuda.get_device_properties(self.dev).multi_processor_count
        if lowrank_sms > 0:
            capi.call("tlora_set_sm_budget", self.device, total - lowrank_sms, lowrank_sms)
        # lowrank_sms < 0: no caps — both streams use full persistent grids and the
        # independent launches fill the SMs freed by each other's ramp-down / tail
        self.side = torch.cuda.Stream(self.dev)
        self.dH = {name: torch.zeros(self.T, lay.R, dtype=torch.bfloat16, device=self.dev)
                   for (L, name), lay in self.layers.items() if L == 0}
        self.overlap = True

    def _ev(self, stream):
        e = torch.cuda.Event()
        e.record(stream)
        return e

    def forward_overlapped(self, main):
        side = self.side
        side.wait_event(self._ev(main))  # adapters of the previous optimizer step are final
        ready = []
        for L, name in self.keys:  # all shrinks run ahead on the side stream
            self.layers[(L, name)].shrink(self.plans[name], self.x_of(name), self.H[(L, name)],
                                          stream=side)
            ready.append(self._ev(side))
        for (L, name), ev in zip(self.keys, ready):
            main.wait_event(ev)
            self.layers[(L, name)].fused_gemm(self.plans[name], self.x_of(name),
                                              self.H[(L, name)], self.Y[name], stream=main)

    def backward_overlapped(self, main, on_layer_done=None):
        """dH of the next projection is computed ahead on the side stream, so the main
        stream's dX never waits behind the previous projection's dA / dB."""
        side = self.side
        side.wait_event(self._ev(main))
        keys = list(reversed(self.keys))
        last_dx = {}  # projection name -> event of the last dX that read dH[name]

        def launch_dh(i):
            L, name = keys[i]
            if name in last_dx:  # dH[name] is shared by every layer of this projection
                side.wait_event(last_dx[name])  # (its grad_a reader is earlier on `side`)
            self.layers[keys[i]].dh(self.plans[name], self.dy_of(name), self.dH[name], stream=side)
            return self._ev(side)

        ev_dh = launch_dh(0)
        for i, (L, name) in enumerate(keys):
            lay, pl = self.layers[(L, name)], self.plans[name]
            main.wait_event(ev_dh)
            lay.dx(pl, self.dy_of(name), self.dH[name], self.dX[name], stream=main)
            last_dx[name] = self._ev(main)
            nxt = i + 1 < len(keys)
            ahead = nxt and keys[i + 1][1] != name
            ev_dh = launch_dh(i + 1) if ahead else None
            lay.grad_b(pl, self.H[(L, name)], self.dy_of(name), stream=side)
            lay.grad_a(pl, self.x_of(name), self.dH[name], stream=side)
            ev_grads = self._ev(side)
            if nxt and not ahead:
                ev_dh = launch_dh(i + 1)
            if on_layer_done is not None:
                on_layer_done((L, name), lay, ev_grads)
        main.wait_stream(side)

    def enable_optimizer(self, base_lr: float = 1e-4, weight_decay: float = 0.01):
        """Per-job AdamW hyperparameters (each job is an independent fine-tuning run)."""
        lrs = [base_lr * (1.0 + 0.25 * (s % 4)) for s in range(len(self.wl.jobs))]
        for lay in self.layers.values():
            lay.set_optimizer(lrs, weight_decay)
        self.optim = True

    def optimizer_step(self, stream=None, grad_scale: float = 1.0):
        for lay in self.layers.values():
            lay.optimizer_step(grad_scale, stream=stream)

    def capture(self, warmup: int = 1, profile: bool = False):
        """Capture one training step (fwd + bwd + AdamW) into a CUDA graph. All launches are
        enqueue-only with device-side state (tile tables, optimizer step counters), so the
        graph replays a fresh step each time; workspaces are sized by the eager warm-up."""
        for _ in range(warmup):
            self.step()
        torch.cuda.synchronize(self.dev)
        from . import capi
        g = torch.cuda.CUDAGraph()
        n0 = capi.lib().tlora_launch_count()
        if profile:  # per-launch CUDA-event brackets become event-record nodes of the graph:
            capi.call("tlora_profile_begin")  # every replay re-records them
        with torch.cuda.graph(g):
            self.step()
        self.graph_launches = capi.lib().tlora_launch_count() - n0  # kernels per replay
        self.graph = g
        return g

    def step(self, stream=None, on_layer_done=None):
        """One training step: forward, backward, fused AdamW update of every adapter. With
        side-stream gradients and no cross-replica exchange, each projection's AdamW runs
        on the side stream right after its dB+dA (overlapping the remaining GEMMs)."""
        self.forward(stream)
        self.backward_and_update(stream, on_layer_done)

    def backward_and_update(self, stream=None, on_layer_done=None, grad_scale: float = 1.0):
        optim = getattr(self, "optim", False)
        inline = (optim and on_layer_done is None and grad_scale == 1.0 and self.chain
                  and getattr(self, "side_grads", False))
        if inline:
            self.backward_chained(stream, opt_inline=True)
            return
        self.backward(stream, on_layer_done=on_layer_done)
        if optim:
            self.optimizer_step(stream, grad_scale)

    def input_tensors(self):
        """Every tensor a step reads from outside the layer (for the e2e host copies)."""
        return list(self.X.values()) + list(self.dY.values())

    # ---- double-buffered inputs (e2e: H2D of step i+1 overlaps compute of step i)
    def make_input_sets(self, n: int = 2):
        self._sets = [(self.X, self.dY)]
        for _ in range(n - 1):
            self._sets.append(({g: t.clone() for g, t in self.X.items()},
                               {p: t.clone() for p, t in self.dY.items()}))
        return [list(X.values()) + list(dY.values()) for X, dY in self._sets]

    def use_inputs(self, i: int):
        self.X, self.dY = self._sets[i]
