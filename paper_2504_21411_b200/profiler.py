"""B200 profiler: measures this box and writes the planner's profile JSON.

The reference ingests profiles (SPEC.md:8 puts measurement out of scope); this module
is the paper's "Profiler" for B200, writing exactly the reference
schema (profiles.py:233-422) so the unchanged search consumes it:

* ``device_flops``: the *effective* rate at which the runtime executes a decoder
  layer's cost-model FLOPs.  One layer of the target model is run fwd+bwd on galv
  kernels at the given microbatch, and device_flops = 3 * fwd_flops / t(fwd+bwd),
  with fwd_flops = flops_per_token * t + flops_per_token_sq * b * s^2 exactly as the
  cost model counts them (costmodel.py:104-106).  Calibration happens only through
  this profile input; the cost model itself is unchanged.
* ``bandwidth_table``: NCCL bus bandwidth per group size g (all-reduce busbw
  convention 2(g-1)/g * V / t, all-gather (g-1)/g * V / t; the table keeps the
  smaller of the two so the model's ring passes are not optimistic) and an alpha fitted
  from a small message so lat*(g-1) reproduces it (collectives.py:49-57).
  Requires torchrun with >= 2 ranks; on one GPU the table is left to the caller.
* ``device_memory_bytes``: total HBM; ``memory_reserve_fraction`` covers the CUDA
  context, allocator fragmentation, logits and transient buffers the model ignores.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import torch
import torch.distributed as dist

from .planner import profiles as P
from .planner.strategy import ParallelStrategy


def _time_cuda(fn, iters: int = 5, warmup: int = 2) -> float:
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters / 1e3


def measure_layer_flops(cfg, microbatch: int, *, iters: int = 3, sustain_s: float = 6.0) -> dict:
    """Effective FLOP/s of one decoder layer fwd+bwd (tp=1, dp=1) on this GPU."""
    from .runtime.config import HybridConfig, profile_for
    from .runtime.layers import DecoderLayer
    from .runtime.topology import Topology
    one = cfg.with_(n_layers=1)
    s = ParallelStrategy(1, 1, 0, False, False)
    hc = HybridConfig(pp=1, microbatch=microbatch, n_microbatches=1, stage_ranges=((0, 1),),
                      layer_strategies=(s,))
    topo = Topology(hc, rank=0, world=1)
    dev = torch.device("cuda", torch.cuda.current_device())
    layer = DecoderLayer(one, 0, s, topo, dtype=torch.bfloat16, grad_dtype=torch.bfloat16,
                         device=dev)
    from .runtime.init import layer_param_shapes
    gen = torch.Generator(device=dev)
    gen.manual_seed(0)
    layer.store.load({n: 0.02 * torch.randn(shp, generator=gen, device=dev)
                      if not n.endswith("norm.weight") else torch.ones(shp, device=dev)
                      for n, shp in layer_param_shapes(one).items()})
    T = microbatch * cfg.seq_len
    x = torch.randn(T, cfg.hidden, device=dev, dtype=torch.bfloat16)
    dy = torch.randn_like(x) * 1e-3

    def step():
        y, ctx = layer.forward(x, microbatch)
        layer.backward(dy, ctx)

    # sustained rate: the GPU runs at ~1 kW cap under a long training step, so time the
    # layer back to back for `sustain_s` seconds and keep the steady-state second half
    for _ in range(2):
        step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n_runs = 0
    while time.perf_counter() - t0 < sustain_s / 2:
        step()
        n_runs += 1
        if n_runs % 4 == 0:
            torch.cuda.synchronize()
    t = _time_cuda(step, iters=max(iters, n_runs), warmup=0)
    lp = profile_for(cfg).layers[0]
    fwd_flops = lp.flops_per_token * T + lp.flops_per_token_sq * microbatch * cfg.seq_len ** 2
    return {"seconds_fwd_bwd": t, "fwd_flops": fwd_flops,
            "device_flops": 3.0 * fwd_flops / t}


def measure_activation_bytes(cfg, microbatch: int) -> dict:
    """Bytes per token one decoder layer keeps alive between its forward and backward
    (tp=1): the allocator delta across ``layer.forward`` with saved state, and with
    recompute (only the boundary tensor survives).  Feeds the cost model's activation
    coefficients (costmodel.py:162-175) instead of the analytic count."""
    from .runtime.config import HybridConfig
    from .runtime.init import layer_param_shapes
    from .runtime.layers import DecoderLayer
    from .runtime.topology import Topology
    one = cfg.with_(n_layers=1)
    dev = torch.device("cuda", torch.cuda.current_device())
    T = microbatch * cfg.seq_len
    out = {}
    for rc in (False, True):
        s = ParallelStrategy(1, 1, 0, False, rc)
        hc = HybridConfig(pp=1, microbatch=microbatch, n_microbatches=1,
                          stage_ranges=((0, 1),), layer_strategies=(s,))
        layer = DecoderLayer(one, 0, s, Topology(hc, rank=0, world=1), dtype=torch.bfloat16,
                             grad_dtype=torch.bfloat16, device=dev)
        layer.store.load({n: 0.02 * torch.ones(shp, device=dev)
                          for n, shp in layer_param_shapes(one).items()})
        x = torch.randn(T, cfg.hidden, device=dev, dtype=torch.bfloat16)
        y, ctx = layer.forward(x, microbatch)  # warm the allocator / tables
        layer.backward(torch.zeros_like(y), ctx)
        del y, ctx
        torch.cuda.synchronize()
        m0 = torch.cuda.memory_allocated()
        y, ctx = layer.forward(x, microbatch)
        torch.cuda.synchronize()
        out["recompute" if rc else "saved"] = (torch.cuda.memory_allocated() - m0) / T
        del y, ctx, layer
        torch.cuda.synchronize()
    return {"bytes_per_token_saved": out["saved"],
            "bytes_per_token_recompute": out["recompute"], "microbatch": microbatch}


def measure_working_set(cfg, microbatch: int) -> dict:
    """Per-token bytes the step holds *beyond* the saved activations at its memory peak
    (tp=1, pp=1): the peak is either the head (logits chunks, cross-entropy stats, dlogits
    -> dx) on top of every layer's saved activations, or the last layer's backward (its
    dy plus the backward temporaries: dgrads, dq|dk|dv, re-gathered inputs) while its own
    saved activations are still alive.  Folded into the last layer's activation term
    (fold_embedding_head) so the unchanged cost model's stage peak covers it."""
    from .runtime.config import HybridConfig
    from .runtime.init import layer_param_shapes
    from .runtime.layers import DecoderLayer, Head
    from .runtime.topology import Topology
    one = cfg.with_(n_layers=1)
    dev = torch.device("cuda", torch.cuda.current_device())
    T = microbatch * cfg.seq_len
    s = ParallelStrategy(1, 1, 0, False, False)
    hc = HybridConfig(pp=1, microbatch=microbatch, n_microbatches=1, stage_ranges=((0, 1),),
                      layer_strategies=(s,))
    topo = Topology(hc, rank=0, world=1)
    kw = dict(dtype=torch.bfloat16, grad_dtype=torch.bfloat16, device=dev)
    layer = DecoderLayer(one, 0, s, topo, **kw)
    layer.store.load({n: 0.02 * torch.ones(shp, device=dev)
                      for n, shp in layer_param_shapes(one).items()})
    x = torch.randn(T, cfg.hidden, device=dev, dtype=torch.bfloat16)
    for _ in range(2):  # the second pass runs with warm allocator / tables / workspaces
        y, ctx = layer.forward(x, microbatch)
        del y
        torch.cuda.synchronize()
        m_saved = torch.cuda.memory_allocated()
        dy = torch.randn_like(x) * 1e-3
        torch.cuda.reset_peak_memory_stats()
        dx = layer.backward(dy, ctx)
        torch.cuda.synchronize()
        layer_ws = torch.cuda.max_memory_allocated() - m_saved  # dy + temporaries (+ dx)
        del dx, ctx, dy
    del layer
    head = Head(cfg, s, topo, **kw)
    head.store.load({n: (0.02 if n == "lm_head.weight" else 1.0) *
                     torch.ones(shp, device=dev) for n, (_, shp) in head.store.layout.items()})
    labels = torch.randint(0, cfg.vocab, (T,), device=dev)
    for _ in range(2):
        torch.cuda.synchronize()
        m0 = torch.cuda.memory_allocated()
        torch.cuda.reset_peak_memory_stats()
        loss, dx = head.forward_backward(x, labels, 1.0 / T)
        torch.cuda.synchronize()
        # logits chunk, stats, dn, dx + the head's input (the last layer's output y, which
        # no layer saves)
        head_ws = torch.cuda.max_memory_allocated() - m0 + x.numel() * x.element_size()
        del loss, dx
    del head
    torch.cuda.synchronize()
    return {"layer_backward_bytes_per_token": layer_ws / T,
            "head_bytes_per_token": head_ws / T,
            "working_set_bytes_per_token": max(layer_ws, head_ws) / T,
            "microbatch": microbatch}


def fold_embedding_head(prof: P.ModelProfile, cfg, working_set_per_token: float = 0.0,
                        first_working_set_per_token: float = 0.0) -> P.ModelProfile:
    """Charge the embedding and the LM head to the planned layers that share their
    strategy (the runtime builds them on layer 0's / layer L-1's tp and dp groups,
    runtime/engine.py): layer 0 gains the embedding tables' parameters, layer L-1 the
    head's parameters and its 2*h*V forward FLOPs per token (backward = 2x fwd by
    costmodel.py:106, i.e. the dgrad + wgrad GEMMs).  The reference has no
    embedding/head layers, so without this the cost model under-predicts
    by the head's share of the step (13% on GPT-2-medium, 9% on GPT-1.3B) and the
    memory prediction misses 16 B/param of vocab tables.  The runtime shards the tables
    with the layer's ZeRO stage too (layers.Embedding / Head), so the fold is exact.

    ``working_set_per_token`` (measure_working_set) is added to the last layer's
    tp-shardable activation bytes: the step's peak is the saved activations plus this
    working set, and the last layer's stage is where it occurs (pp=1: every stage is the
    last; pp>1: the head's stage holds one microbatch in flight).
    ``first_working_set_per_token`` goes to layer 0 the same way: the first pipeline stage
    (pp > 1) peaks in a layer backward too, with no head to carry it (pp = 1 charges both,
    a conservative overlap).  Residual: middle stages of pp >= 3 carry no working set, and
    when the last layer itself recomputes the cost model charges it boundary bytes only."""
    L, h, V = cfg.n_layers, cfg.hidden, cfg.vocab
    emb = V * h + (cfg.seq_len * h if cfg.arch == "gpt" else 0)
    head = V * h + h * (2 if cfg.arch == "gpt" else 1)
    layers = list(prof.layers)

    def bump(lp, params, fpt, ws=0.0):
        return P.LayerProfile(
            param_count=lp.param_count + params, flops_per_token=lp.flops_per_token + fpt,
            flops_per_token_sq=lp.flops_per_token_sq,
            act_shardable_bytes_per_token=lp.act_shardable_bytes_per_token + ws,
            act_replicated_bytes_per_token=lp.act_replicated_bytes_per_token,
            boundary_bytes_per_token=lp.boundary_bytes_per_token)

    layers[0] = bump(layers[0], emb, 0, float(first_working_set_per_token))
    layers[L - 1] = bump(layers[L - 1], head, 2 * h * V, float(working_set_per_token))
    out = P.ModelProfile(n_layers=prof.n_layers, hidden_size=prof.hidden_size,
                         seq_len=prof.seq_len, layers=tuple(layers))
    out.validate()
    return out


def planned_profile(cfg) -> P.ModelProfile:
    """Analytic decoder-layer profile with the embedding/head folded in (fallback when
    no activation-calibrated profile was measured for ``cfg``)."""
    from .runtime.config import profile_for
    return fold_embedding_head(profile_for(cfg), cfg)


def calibrated_model_profile(cfg, act: dict) -> P.ModelProfile:
    """The analytic profile with its activation coefficients scaled to the measured bytes:
    shardable/replicated keep their analytic split; boundary = the recompute residue."""
    from .runtime.config import profile_for
    base = profile_for(cfg)
    lp = base.layers[0]
    analytic = lp.act_shardable_bytes_per_token + lp.act_replicated_bytes_per_token
    f = act["bytes_per_token_saved"] / analytic
    layer = P.LayerProfile(
        param_count=lp.param_count, flops_per_token=lp.flops_per_token,
        flops_per_token_sq=lp.flops_per_token_sq,
        act_shardable_bytes_per_token=lp.act_shardable_bytes_per_token * f,
        act_replicated_bytes_per_token=lp.act_replicated_bytes_per_token * f,
        boundary_bytes_per_token=max(act["bytes_per_token_recompute"],
                                     lp.boundary_bytes_per_token))
    prof = P.ModelProfile(n_layers=base.n_layers, hidden_size=base.hidden_size,
                          seq_len=base.seq_len, layers=(layer,) * base.n_layers)
    prof.validate()
    return fold_embedding_head(
        prof, cfg,
        act.get("working_set_bytes_per_token", 0.0)
        + act.get("step_memory_extra_bytes_per_token", 0.0),
        act.get("layer_backward_bytes_per_token", 0.0)
        + act.get("step_memory_extra_first_bytes_per_token", 0.0))


def step_memory_extra(lines: list) -> dict:
    """Per-token bytes to add to the working-set fold so the cost model's stage peak covers
    what a full training step held on the GPU, from bench.py JSON lines (their "memory"
    object: runtime peak incl. symmetric NVLink allocations vs the plan's predicted stage
    peak).  What the single-layer measurement cannot see lives here: the ZeRO-2 full-size
    gradient ring of the NVLink dp pool, tp peer buffers, the gathered (tp-replicated)
    backward temporaries of Megatron-SP, rope tables.  The excess of a line is charged to
    its last layer's tp-shardable activation term (act = tokens*(shard/tp + ...)):
    extra = excess * tp / (microbatch * seq / dp); the maximum over the lines is kept.
    Lines whose last layer recomputes (the term is not used then) or that are not the
    last pipeline stage are skipped."""
    best, best_first, used, skipped = 0.0, 0.0, [], []
    for ln in lines:
        m = ln.get("memory", {})
        pp, st = m.get("pp", 1), m.get("stage")
        first = pp > 1 and st == 0
        ll = m.get("first_layer" if first else "last_layer")
        if not ll or (st != pp - 1 and not first) or ll.get("recompute"):
            skipped.append(ln.get("config", {}).get("parallelism"))
            continue
        excess = m["runtime_peak_gb"] * 1e9 - m["predicted_gb"] * 1e9
        # the first stage holds min(m, pp) microbatches; its layer-0 fold counts once per
        # microbatch in flight (costmodel.in_flight_microbatches)
        inflight = m.get("in_flight", 1) if first else 1
        tokens = m["microbatch"] * m["seq_len"] / ll["dp"] * inflight
        x = max(excess, 0.0) * ll["tp"] / tokens
        used.append({"config": ln.get("config", {}).get("parallelism"), "n_gpus": ln.get("n_gpus"),
                     "stage": st, "fold": "layer 0" if first else "layer L-1",
                     "excess_bytes": excess, "extra_bytes_per_token": x})
        if first:
            best_first = max(best_first, x)
        else:
            best = max(best, x)
    return {"step_memory_extra_bytes_per_token": best,
            "step_memory_extra_first_bytes_per_token": best_first,
            "step_memory_sources": used, "step_memory_skipped": skipped}


def measure_collectives(sizes=(2 ** 20, 2 ** 24, 2 ** 28)) -> dict:
    """busbw (bytes/s) and alpha per contiguous group size; rank 0 returns the table."""
    world = dist.get_world_size()
    rank = dist.get_rank()
    out = {}
    g = 2
    while g <= world:
        members = [list(range(s, s + g)) for s in range(0, world, g)]
        groups = [dist.new_group(m) for m in members]
        grp = groups[rank // g]
        res = {}
        for nbytes in sizes:
            n = nbytes // 2
            x = torch.ones(n, dtype=torch.bfloat16, device="cuda")
            y = torch.empty(n * 1, dtype=torch.bfloat16, device="cuda")
            t_ar = _time_cuda(lambda: dist.all_reduce(x, group=grp), iters=10)
            chunk = torch.ones(n // g, dtype=torch.bfloat16, device="cuda")
            t_ag = _time_cuda(lambda: dist.all_gather_into_tensor(y, chunk, group=grp), iters=10)
            res[nbytes] = (t_ar, t_ag)
        big = sizes[-1]
        t_ar, t_ag = res[big]
        bw_ar = 2 * (g - 1) / g * big / t_ar
        bw_ag = (g - 1) / g * big / t_ag
        bw = min(bw_ar, bw_ag)
        small_t = res[sizes[0]][1]
        lat = max(small_t - (g - 1) / g * sizes[0] / bw, 0.0) / (g - 1)
        out[g] = {"bus_bandwidth": bw, "latency": lat, "ar_busbw": bw_ar, "ag_busbw": bw_ag}
        g *= 2
    return out


def measure_dp_overlap(cfg, cluster, global_batch: int, *, steps: int = 4,
                       warmup: int = 2, rounds: int = 3) -> dict:
    """Measured ``comm_overlap_fraction`` (reference profiles.py:187, costmodel.py:265,
    search.py:193): how much of the cost model's dp-sync time the runtime hides behind
    compute.  Under torchrun, the searched plan for this world is run twice with the same
    per-rank work -- with its dp collectives (reduce-scatter / all-reduce overlapped with
    the backward, parameter all-gather fused into AdamW) and with them skipped
    (params.SKIP_DP_SYNC, timing only) -- and

        exposed = T_step(sync) - T_step(no sync)        (device time, max over ranks)
        overlap = clamp(1 - exposed / max_stage(dp_sync_time), 0, 1)

    with dp_sync_time the plan's modeled per-stage sync (overlap 0)."""
    from .planner.search import SearchConfig, optimize
    from .runtime import params as params_mod
    from .runtime.config import get_hybrid_parallel_configs
    from .runtime.engine import construct_hybrid_parallel_model
    from .runtime.init import synthetic_tokens
    model_prof = load_or_plan_profile(cfg)
    training = P.TrainingConfig(global_batch=global_batch)
    plan = optimize(model_prof, cluster, training, SearchConfig())
    hc = get_hybrid_parallel_configs(plan, cfg)
    model = construct_hybrid_parallel_model(cfg, hc, training=training, dtype=torch.bfloat16,
                                            init="fast")
    tokens = synthetic_tokens(cfg, global_batch).cuda()

    def timed() -> float:
        for _ in range(warmup):
            model.train_step(tokens)
        model.wait_optimizer()
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(steps):
            model.train_step(tokens)
        model.wait_optimizer()
        b.record()
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / steps / 1e3], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    # alternate the two variants (clock / power drift hits both alike), median of each
    syncs, nosyncs = [], []
    try:
        for _ in range(rounds):
            params_mod.SKIP_DP_SYNC = False
            syncs.append(timed())
            params_mod.SKIP_DP_SYNC = True
            nosyncs.append(timed())
    finally:
        params_mod.SKIP_DP_SYNC = False
    import statistics
    t_sync, t_nosync = statistics.median(syncs), statistics.median(nosyncs)
    modeled = max(c.dp_sync_time for c in plan.cost_breakdown)
    exposed = t_sync - t_nosync
    overlap = min(max(1.0 - exposed / modeled, 0.0), 1.0) if modeled > 0 else 0.0
    return {"t_step_sync_s": t_sync, "t_step_nosync_s": t_nosync, "exposed_s": exposed,
            "samples_sync_s": syncs, "samples_nosync_s": nosyncs,
            "modeled_dp_sync_s": modeled, "comm_overlap_fraction": overlap,
            "plan": [s.to_dict() for s in plan.layer_strategies[:1]],
            "plan_microbatch": plan.microbatch, "world": dist.get_world_size()}


def load_or_plan_profile(cfg) -> P.ModelProfile:
    """The committed activation-calibrated model profile, else the analytic one."""
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "profiles", f"b200_model_{cfg.name}.json")
    if os.path.exists(path):
        return P.load_model_profile(path)
    return planned_profile(cfg)


def build_cluster(n_devices: int, device_flops: float, table: dict, *,
                  reserve: float = 0.1, memory: int | None = None) -> P.ClusterProfile:
    mem = memory if memory is not None else (
        torch.cuda.get_device_properties(0).total_memory if torch.cuda.is_available()
        else 180_000_000_000)
    entries = tuple(P.BandwidthEntry("intra_node", g, v["bus_bandwidth"], v["latency"])
                    for g, v in sorted(table.items()))
    c = P.ClusterProfile(n_devices, min(n_devices, 8), float(device_flops), int(mem), reserve,
                         entries)
    c.validate()
    return c


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="galv-profile")
    ap.add_argument("-o", "--output", required=True)
    ap.add_argument("--model", default="llama2-7b")
    ap.add_argument("--microbatch", type=int, default=2)
    ap.add_argument("--devices", type=int, default=8, help="n_devices written to the profile")
    ap.add_argument("--reserve", type=float, default=0.1)
    ap.add_argument("--device-memory", type=int, default=None,
                    help="device_memory_bytes to write (default: this GPU's total HBM); "
                         "BASELINE C5 plans under 180e9 with --reserve 0")
    ap.add_argument("--flops-from", default=None,
                    help="reuse device_flops of this cluster profile (skip the layer timing)")
    ap.add_argument("--table-from", default=None, help="reuse the bandwidth table of a profile")
    ap.add_argument("--model-out", default=None,
                    help="also write the activation-calibrated ModelProfile of --model here")
    ap.add_argument("--overlap-out", default=None,
                    help="under torchrun: measure comm_overlap_fraction of the searched "
                         "plan for --model at this world size (--cluster-in) and write a "
                         "TrainingConfig JSON here")
    ap.add_argument("--cluster-in", default=None, help="cluster profile for --overlap-out")
    ap.add_argument("--seqs-per-gpu", type=int, default=8)
    ap.add_argument("--memory-from", nargs="+", default=None,
                    help="bench.py JSON lines of --model: fold the measured step-memory excess "
                         "over the prediction into --model-out (step_memory_extra)")
    ap.add_argument("--skip-flops", action="store_true",
                    help="with --table-from + --model-out: only measure activations")
    args = ap.parse_args(argv)
    from .runtime.config import MODEL_PRESETS
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if torch.cuda.is_available():
        torch.cuda.set_device(local)
    table = {}
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        if not args.overlap_out:
            table = measure_collectives()
    elif args.table_from:
        c = P.load_cluster_profile(args.table_from)
        table = {e.group_size: {"bus_bandwidth": e.bus_bandwidth, "latency": e.latency}
                 for e in c.bandwidth_table if e.span == "intra_node"}
    rank = dist.get_rank() if world > 1 else 0
    if args.memory_from:
        # offline: rewrite --model-out's profile with the step-memory calibration folded in
        cfg = MODEL_PRESETS[args.model]
        meta_path = os.path.splitext(args.model_out)[0] + ".meta.json"
        with open(meta_path) as fh:
            meta = json.load(fh)
        lines = []
        for path in args.memory_from:
            with open(path) as fh:
                for raw in fh:
                    raw = raw.strip()
                    if raw.startswith("{") and '"memory"' in raw:
                        d = json.loads(raw)
                        if d.get("config", {}).get("model") == cfg.name:
                            lines.append(d)
        new = step_memory_extra(lines)
        act = meta["activation"]
        # a fold without new measurements keeps its previous calibration (the lines of an
        # earlier bench generation were measured against a profile without the extra)
        for key, fold in (("step_memory_extra_bytes_per_token", "layer L-1"),
                          ("step_memory_extra_first_bytes_per_token", "layer 0")):
            if any(src["fold"] == fold for src in new["step_memory_sources"]):
                act[key] = new[key]
        act["step_memory_sources"] = [s for s in act.get("step_memory_sources", [])
                                      if s.get("fold", "layer L-1") not in
                                      {x["fold"] for x in new["step_memory_sources"]}]
        act["step_memory_sources"] += new["step_memory_sources"]
        act["step_memory_skipped"] = new["step_memory_skipped"]
        P.save_profiles(args.model_out, model=calibrated_model_profile(cfg, meta["activation"]))
        with open(meta_path, "w") as fh:
            json.dump(meta, fh, indent=1)
        print(json.dumps({k: meta["activation"][k] for k in meta["activation"]
                          if k.startswith("step_memory")}))
        return 0
    if args.overlap_out:
        if world < 2:
            raise SystemExit("--overlap-out needs torchrun with >= 2 ranks")
        c = P.load_cluster_profile(args.cluster_in)
        table = tuple(e for e in c.bandwidth_table if e.group_size <= world)
        c = P.ClusterProfile(world, min(c.devices_per_node, world), c.device_flops,
                             c.device_memory_bytes, c.memory_reserve_fraction, table)
        gb = args.seqs_per_gpu * world
        res = measure_dp_overlap(MODEL_PRESETS[args.model], c, gb)
        if rank == 0:
            P.save_profiles(args.overlap_out, training=P.TrainingConfig(
                global_batch=gb, comm_overlap_fraction=res["comm_overlap_fraction"]))
            with open(os.path.splitext(args.overlap_out)[0] + ".meta.json", "w") as fh:
                json.dump({"model": args.model, "cluster": args.cluster_in, **res}, fh,
                          indent=1)
            print(json.dumps(res))
        dist.barrier()
        dist.destroy_process_group()
        return 0
    if rank == 0 and args.model_out:
        cfg = MODEL_PRESETS[args.model]
        act = measure_activation_bytes(cfg, args.microbatch)
        act.update(measure_working_set(cfg, args.microbatch))
        # re-measuring activations keeps an existing step-memory calibration
        old = os.path.splitext(args.model_out)[0] + ".meta.json"
        if os.path.exists(old):
            with open(old) as fh:
                prev = json.load(fh).get("activation", {})
            act.update({k: v for k, v in prev.items() if k.startswith("step_memory")})
        P.save_profiles(args.model_out, model=calibrated_model_profile(cfg, act))
        with open(os.path.splitext(args.model_out)[0] + ".meta.json", "w") as fh:
            json.dump({"model": args.model, "activation": act}, fh, indent=1)
        print(json.dumps({"activation": act}))
        if args.skip_flops:
            return 0
    if rank == 0:
        if args.flops_from:
            lay = {"device_flops": P.load_cluster_profile(args.flops_from).device_flops,
                   "from": args.flops_from}
        else:
            lay = measure_layer_flops(MODEL_PRESETS[args.model], args.microbatch)
        if not table:  # single GPU: NVLink table from the pool's published measurements
            table = {g: {"bus_bandwidth": 725e9, "latency": 5e-6} for g in (2, 4, 8)}
        cluster = build_cluster(args.devices, lay["device_flops"], table, reserve=args.reserve,
                                memory=args.device_memory)
        P.save_profiles(args.output, cluster=cluster)
        meta = {"layer": lay, "table": {str(k): v for k, v in table.items()},
                "model": args.model, "microbatch": args.microbatch, "world": world,
                "device_memory_bytes": cluster.device_memory_bytes,
                "memory_reserve_fraction": cluster.memory_reserve_fraction}
        with open(os.path.splitext(args.output)[0] + ".meta.json", "w") as fh:
            json.dump(meta, fh, indent=1)
        print(json.dumps(meta))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_profile_cli(args) -> int:
    """``hybridplan profile`` -> measure this GPU (and NCCL when under torchrun)."""
    return main(["-o", args.output, "--model", {"llama": "llama2-7b", "gpt": "gpt2-medium"}
                 [args.arch], "--devices", str(args.devices)])


if __name__ == "__main__":
    sys.exit(main())
