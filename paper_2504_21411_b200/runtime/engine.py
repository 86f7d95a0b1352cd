"""construct_hybrid_parallel_model + the training step (1F1B pipeline over stages).

One process per GPU (torchrun); ``HybridParallelModel`` owns this rank's stage:
embedding (stage 0), decoder layers of ``stage_ranges[stage]``, head (last stage).
``train_step`` executes the reference's 1F1B op order (pipesim.py:73-82) with NCCL
point-to-point between stages (combined send/recv when a forward is followed by a
backward, as Megatron does, so the rings never deadlock), reshards between layers whose
(tp, dp, sp) differ, synchronizes gradients per ZeRO stage and runs the fused AdamW.
The measured per-op timeline can be exported in the simulator's JSONL trace schema
(pipesim.py:34-49, 264-269) for a measured-vs-simulated diff.
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass

import torch
import torch.distributed as dist

from ..planner.pipesim import SimEvent, one_f_one_b_order
from ..planner.profiles import TrainingConfig
from . import comm
from .config import HybridConfig, ModelConfig
from .init import init_tensor, param_shapes
from .layers import DecoderLayer, Embedding, Head, tp_slice
from . import dp_nvlink
from .reshard import Layout, Resharder
from .topology import Topology


@dataclass(frozen=True)
class OptimConfig:
    lr: float = 3e-4
    beta1: float = 0.9
    beta2: float = 0.95
    eps: float = 1e-8
    weight_decay: float = 0.1


class HybridParallelModel:
    def __init__(self, cfg: ModelConfig, hc: HybridConfig, *, training: TrainingConfig | None = None,
                 dtype=torch.bfloat16, device=None, seed: int = 1234, init: str = "exact",
                 perturb: bool = False, optim: OptimConfig = OptimConfig(), weights=None):
        cfg.validate()
        hc.validate(cfg)
        self.cfg, self.hc, self.dtype = cfg, hc, dtype
        self.training = training or TrainingConfig(global_batch=hc.global_batch)
        self.optim = optim
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.topo = Topology(hc)
        self.stage = self.topo.stage
        self.first = self.stage == 0
        self.last = self.stage == hc.pp - 1
        gdt = torch.float32 if self.training.bytes_per_grad >= 4 else dtype
        lo, hi = hc.stage_ranges[self.stage]
        self.layer_ids = list(range(lo, hi))
        kw = dict(dtype=dtype, grad_dtype=gdt, device=self.device)
        self.layers = [DecoderLayer(cfg, i, hc.layer_strategies[i], self.topo, **kw)
                       for i in self.layer_ids]
        self.embed = Embedding(cfg, hc.layer_strategies[0], self.topo, **kw) if self.first else None
        self.head = Head(cfg, hc.layer_strategies[-1], self.topo, **kw) if self.last else None
        self.resharder = Resharder(self.topo.stage_group, self.topo.local, self.device)
        self.step_count = 0
        self._opt_stream = None
        self.trace: list = []
        self.record_trace = False
        # per-layer CUDA events (report.measured_report): (kind, layer, mb, start, end)
        self.layer_events: list = []
        self.record_layers = False
        self._init_params(seed, init, perturb, weights)
        self.dropout_step = 0  # attention-dropout Philox counter: advanced per train_step
        for layer in self.layers:
            layer.dropout_seed = seed
        # dp collectives of bf16 ZeRO-0/1/2 stores over NVLink/NVSwitch (symmetric pools)
        self.dp_pools = dp_nvlink.attach([st for _, st, _ in self.stores()], self.device)

    # ------------------------------------------------------------------ init
    def stores(self):
        """[(name prefix, ParamStore, owner module)] for this rank's stage."""
        out = []
        if self.embed:
            out.append(("", self.embed.store, self.embed))
        out += [(l.param_prefix(), l.store, l) for l in self.layers]
        if self.head:
            out.append(("", self.head.store, self.head))
        return out

    def _init_params(self, seed, mode, perturb, weights):
        cfg = self.cfg
        for prefix, store, owner in self.stores():
            tp, r = getattr(owner, "wtp", owner.tp), getattr(owner, "wtpr", owner.tpr)
            local = {}
            for name, (_, shape) in store.layout.items():
                full_name = prefix + name
                if weights is not None:
                    full = weights[full_name]
                    local[name] = tp_slice(cfg, full_name, full, tp, r)
                elif mode == "exact":
                    full = init_tensor(full_name, param_shapes(cfg)[full_name], seed=seed,
                                       perturb=perturb)
                    local[name] = tp_slice(cfg, full_name, full, tp, r)
                else:  # "fast": draw the local shard directly on the device
                    local[name] = init_tensor(f"{full_name}@tp{tp}.{r}", shape, seed=seed,
                                              perturb=perturb, device=self.device)
            store.load(local)

    # ------------------------------------------------------------------ data
    def _replica_slice(self, strategy, mb_tokens):
        """Sample range of this rank's dp replica within a microbatch."""
        g = self.topo.dp(strategy.tp)
        per = self.hc.microbatch // strategy.dp
        return g.index * per, (g.index + 1) * per

    def _layout(self, li):
        return Layout.of(self.hc.layer_strategies[li])

    # ------------------------------------------------------------------ forward / backward
    def _fwd(self, k, x_in, tokens):
        """Forward of microbatch k through this stage; returns (output, saved ctx)."""
        cfg, hc = self.cfg, self.hc
        S = cfg.seq_len
        T = hc.microbatch * S
        rec = {"ctxs": [], "mb": k}
        if self.first:
            s0 = hc.layer_strategies[0]
            a, b = self._replica_slice(s0, T)
            ids = tokens[k, a:b, :S].reshape(-1)
            rec["ids"] = ids
            ev = self._ev_start()
            x = self.embed.forward(ids)
            self._ev_end(ev, "embed_fwd", 0, k)
        else:
            x = x_in
        prev = None
        for idx, layer in enumerate(self.layers):
            if idx + 1 < len(self.layers):
                self.layers[idx + 1].store.prefetch()
            lay = Layout.of(layer.s)
            if prev is not None and prev != lay:
                ev = self._ev_start()
                x = self.resharder(x, prev, lay, T)
                self._ev_end(ev, "transition_fwd", layer.index, k)
                rec["ctxs"].append(("reshard", prev, lay))
            B = hc.microbatch // layer.s.dp
            b0 = k * hc.microbatch + self._replica_slice(layer.s, T)[0]
            ev = self._ev_start()
            x, ctx = layer.forward(x, B, b0)
            self._ev_end(ev, "fwd", layer.index, k)
            rec["ctxs"].append(("layer", layer, ctx))
            prev = lay
        if not self.last:
            nxt = self._layout(hc.stage_ranges[self.stage + 1][0])
            if nxt != prev:
                x = self.resharder(x, prev, nxt, T)
                rec["ctxs"].append(("reshard", prev, nxt))
            return x, rec
        sl = hc.layer_strategies[-1]
        a, b = self._replica_slice(sl, T)
        labels = tokens[k, a:b, 1:S + 1].reshape(-1)
        scale = 1.0 / (hc.global_batch * S)
        ev = self._ev_start()
        loss_sum, dx = self.head.forward_backward(x, labels, scale)
        self._ev_end(ev, "head", self.cfg.n_layers - 1, k)
        rec["head_dx"] = dx
        rec["loss"] = loss_sum
        return None, rec

    def _bwd(self, rec, dy):
        T = self.hc.microbatch * self.cfg.seq_len
        dx = rec.pop("head_dx") if self.last else dy
        items = list(reversed(rec["ctxs"]))
        layer_items = [it for it in items if it[0] == "layer"]
        if layer_items:
            layer_items[0][1].store.prefetch()
        nxt_layer = {id(a[1]): b[1] for a, b in zip(layer_items, layer_items[1:])}
        last = -1
        for item in items:
            if item[0] == "layer" and id(item[1]) in nxt_layer:
                nxt_layer[id(item[1])].store.prefetch()
            if item[0] == "reshard":
                _, src, dst = item
                ev = self._ev_start()
                dx = self.resharder(dx, dst, src, T)
                # the transition into layer `last` (recorded under that layer, as in fwd)
                self._ev_end(ev, "transition_bwd", last, rec.get("mb", -1))
            else:
                _, layer, ctx = item
                ev = self._ev_start()
                dx = layer.backward(dx, ctx)
                self._ev_end(ev, "bwd", layer.index, rec.get("mb", -1))
                last = layer.index
        rec["ctxs"] = []
        if self.first:
            ev = self._ev_start()
            self.embed.backward(rec["ids"], dx)
            self._ev_end(ev, "embed_bwd", 0, rec.get("mb", -1))
            return None
        return dx

    # ------------------------------------------------------------------ p2p
    def _p2p(self, ops):
        reqs = dist.batch_isend_irecv(ops) if ops else []
        for r in reqs:
            r.wait()

    def _act_shape(self, li):
        T = self.hc.microbatch * self.cfg.seq_len
        lo, hi = self._layout(li).token_range(self.topo.local, T)
        return (hi - lo, self.cfg.hidden)

    def train_step(self, tokens, *, step_optimizer: bool = True) -> float:
        """One iteration over the global batch. tokens: [GB, S+1] int64 (host or device)."""
        hc, cfg = self.hc, self.cfg
        m = hc.n_microbatches
        tok = tokens.to(self.device, non_blocking=True).view(m, hc.microbatch, cfg.seq_len + 1)
        ops = one_f_one_b_order(hc.pp, self.stage, m)
        for layer in self.layers:
            layer.dropout_step = self.dropout_step
        recs, inputs, grads = {}, {}, {}
        first_layer = hc.stage_ranges[self.stage][0]
        prev_rank, next_rank = self.topo.prev_stage_rank(), self.topo.next_stage_rank()
        in_shape = self._act_shape(first_layer)
        out_shape = (self._act_shape(hc.stage_ranges[self.stage + 1][0])
                     if not self.last else None)
        loss_acc = torch.zeros((), dtype=torch.float32, device=self.device)
        t0 = time.perf_counter()

        def recv_fwd(k):
            buf = torch.empty(in_shape, dtype=self.dtype, device=self.device)
            return buf, dist.P2POp(dist.irecv, buf, prev_rank)

        def recv_bwd(k):
            buf = torch.empty(out_shape, dtype=self.dtype, device=self.device)
            return buf, dist.P2POp(dist.irecv, buf, next_rank)

        for pos, (kind, k1) in enumerate(ops):
            k = k1 - 1
            nxt = ops[pos + 1] if pos + 1 < len(ops) else None
            if kind == "fwd":
                if not self.first and k not in inputs:
                    buf, op = recv_fwd(k)
                    self._p2p([op])
                    inputs[k] = buf
                self._mark("fwd", k1)
                y, rec = self._fwd(k, inputs.pop(k, None), tok)
                recs[k] = rec
                if self.last:
                    loss_acc += rec.pop("loss")
                else:
                    p2p = [dist.P2POp(dist.isend, y.contiguous(), next_rank)]
                    if nxt is not None and nxt[0] == "bwd":
                        buf, op = recv_bwd(nxt[1] - 1)
                        p2p.append(op)
                        grads[nxt[1] - 1] = buf
                    self._p2p(p2p)
            else:
                if k1 == m:  # last microbatch: layers launch their dp sync as they finish
                    for _, store, _ in self.stores():
                        store.last_window = True
                if not self.last and k not in grads:
                    buf, op = recv_bwd(k)
                    self._p2p([op])
                    grads[k] = buf
                self._mark("bwd", k1)
                dx = self._bwd(recs.pop(k), grads.pop(k, None))
                if not self.first:
                    p2p = [dist.P2POp(dist.isend, dx.contiguous(), prev_rank)]
                    if nxt is not None and nxt[0] == "fwd":
                        buf, op = recv_fwd(nxt[1] - 1)
                        p2p.append(op)
                        inputs[nxt[1] - 1] = buf
                    self._p2p(p2p)
        self._mark("dp_sync", -1)
        self._sync_grads()
        if step_optimizer:
            self._optimizer_step()
        self._mark("end", -1)
        # loss: sum over dp replicas of the last stage, counted once per replica (tp rank 0)
        if self.topo.distributed:
            if not (self.last and self.head.tpg.index == 0):
                loss_acc.zero_()
            dist.all_reduce(loss_acc)
        self.last_step_time = time.perf_counter() - t0
        self.dropout_step += 1
        return loss_acc / (hc.global_batch * cfg.seq_len)

    def _ev_start(self):
        if not self.record_layers:
            return None
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        return ev

    def _ev_end(self, start, kind, layer, mb):
        if start is None:
            return
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        self.layer_events.append((kind, layer, mb, start, ev))

    def layer_times(self) -> list:
        """[(kind, layer, microbatch, seconds)] of the recorded layer events."""
        torch.cuda.synchronize()
        return [(k, li, mb, a.elapsed_time(b) / 1e3) for k, li, mb, a, b in self.layer_events]

    def _mark(self, kind, mb):
        if self.record_trace:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            self.trace.append((kind, mb, ev))

    def measured_trace(self) -> list:
        """Recorded ops as SimEvents (seconds since the first mark), pipesim schema."""
        if not self.trace:
            return []
        torch.cuda.synchronize()
        t0 = self.trace[0][2]
        out = []
        for (kind, mb, ev), nxt in zip(self.trace, self.trace[1:]):
            if kind == "end":
                continue
            start = t0.elapsed_time(ev) / 1e3
            dur = ev.elapsed_time(nxt[2]) / 1e3
            out.append(SimEvent(time=start, device_stage=self.stage, kind=kind,
                                microbatch_id=mb, duration=dur))
        return out

    # ------------------------------------------------------------------ sync + optimizer
    def _sync_grads(self):
        for _, store, _ in self.stores():
            store.sync()

    def _optimizer_step(self):
        """Fused AdamW per store on a side stream: the HBM-bound update of layer i overlaps
        the next step's forward of layers < i (each store's next use waits on its event)."""
        self.step_count += 1
        o = self.optim
        if os.environ.get("GALV_OPT_SIDE_STREAM", "1") == "0":  # A/B: serial optimizer
            for _, store, _ in self.stores():
                store.step(lr=o.lr, beta1=o.beta1, beta2=o.beta2, eps=o.eps,
                           weight_decay=o.weight_decay, step=self.step_count)
                store.zero_grads()
            return
        if self._opt_stream is None:
            self._opt_stream = torch.cuda.Stream(device=self.device)
        done = torch.cuda.Event()
        done.record()
        self._opt_stream.wait_event(done)
        with torch.cuda.stream(self._opt_stream):
            for _, store, _ in self.stores():
                store.step(lr=o.lr, beta1=o.beta1, beta2=o.beta2, eps=o.eps,
                           weight_decay=o.weight_decay, step=self.step_count)
                store.zero_grads()
                ev = torch.cuda.Event()
                ev.record()
                store.ready_event = ev

    def symmetric_bytes(self) -> int:
        """Device memory in symmetric (NVLink) allocations, outside the caching allocator:
        the dp pools of this model and the tp peer buffers."""
        from . import nvlink
        return sum(p.nbytes for p in self.dp_pools) + nvlink.symmetric_bytes()

    def wait_optimizer(self):
        """Make the current stream wait for the optimizer side stream (timing edges)."""
        if self._opt_stream is not None:
            torch.cuda.current_stream().wait_stream(self._opt_stream)

    def zero_grads(self):
        for _, store, _ in self.stores():
            store.zero_grads()

    # ------------------------------------------------------------------ tests / export
    def full_gradients(self) -> dict:
        """Logical (unsharded) gradients of this stage's params; collective over the stage."""
        from .layers import tp_unslice
        out = {}
        for prefix, store, owner in self.stores():
            flat = store.full_grad()[:store.total]
            views = store.views(flat)
            for name, v in views.items():
                parts = [v]
                if getattr(owner, "wtp", owner.tp) > 1:
                    g = torch.empty((owner.tp,) + tuple(v.shape), dtype=v.dtype, device=v.device)
                    dist.all_gather_into_tensor(g, v.contiguous(), group=owner.tpg.group)
                    parts = list(g.unbind(0))
                out[prefix + name] = tp_unslice(self.cfg, prefix + name, parts)
        return out

    def memory_report(self) -> dict:
        tot = {"param": 0, "grad": 0, "optimizer": 0}
        for _, store, _ in self.stores():
            for k, v in store.memory_bytes().items():
                tot[k] += v
        return tot


def construct_hybrid_parallel_model(model_cfg: ModelConfig, hybrid_config: HybridConfig,
                                    **kw) -> HybridParallelModel:
    """Paper entry point: build this rank's share of the hybrid model."""
    return HybridParallelModel(model_cfg, hybrid_config, **kw)
