#!/usr/bin/env python
"""Training-throughput benchmark: the searched hybrid plan for Llama-2-7B on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl galv|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Metric (BASELINE.json): Llama-2-7B train tokens/s (whole job), MFU vs 2.25 PF/GPU dense
bf16, and the cost model's predicted vs the measured iteration time.  A "step" is one
optimizer iteration over a global batch of 8*N sequences of 4096 synthetic tokens
(random-init weights), executed by the plan the planner picks for N B200s.

``value`` times K steps with the tokens already in HBM (CUDA events, barrier +
synchronize on both sides, max over ranks); ``e2e`` times K more steps through the
public API with the tokens in pinned host memory (H2D inside the step) and the loss
read back to the host every step.  ``--impl reference`` times the CPU restatement
(oracle/, the only CPU implementation of this path: the reference repository has no
training code) on the host cores and prints the same JSON line.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAK_BF16_DENSE = 2.25e15


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("galv", "reference"), default="galv")
    ap.add_argument("--model", default="llama2-7b")
    ap.add_argument("--seqs-per-gpu", type=int, default=8)
    ap.add_argument("--cluster-profile", default=None,
                    help="default: the profile calibrated on --model's layer "
                         "(CLUSTER_PROFILES), else profiles/b200_cluster.json")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--plan-out", default=None)
    ap.add_argument("--trace-out", default=None,
                    help="write the measured step timeline (pipesim JSONL schema) + sim diff")
    ap.add_argument("--report-out", default=None,
                    help="write the measured-vs-predicted per-layer/per-stage report "
                         "(reference build_report bundle + measured columns) to PATH.json/.csv")
    ap.add_argument("--layer-pattern", default=None,
                    help="explicit per-layer strategies instead of the search, cycled over "
                         "layers, e.g. 'tp8,dp8z3,tp4dp2' (BASELINE config 4)")
    ap.add_argument("--microbatch", type=int, default=None, help="with --layer-pattern")
    ap.add_argument("--pp", type=int, default=1,
                    help="with --layer-pattern: pipeline stages (strategies cover n/pp GPUs)")
    ap.add_argument("--sp-mode", choices=("megatron", "ulysses"), default="megatron",
                    help="how sp=True layers run: Megatron-SP or DeepSpeed-Ulysses")
    return ap.parse_args()


# ----------------------------------------------------------------------------- helpers


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return d, "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, \
            "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# cluster profiles calibrated on each model's own layer (profiles/*.meta.json); llama2-13b's
# at seq 32K (config C5), gpt2-medium's at seq 1024 (C2); everything else uses the 7B one
CLUSTER_PROFILES = {"llama2-13b": "b200_cluster_llama13b_180g.json",  # C5: 180e9, reserve 0
                    "gpt2-medium": "b200_cluster_gpt2m.json"}


def default_cluster_profile(model: str) -> str:
    return os.path.join(ROOT, "profiles", CLUSTER_PROFILES.get(model, "b200_cluster.json"))


def cluster_profile(n: int, path: str):
    from paper_2504_21411_b200.planner import profiles as P
    shown = os.path.relpath(path, ROOT) if os.path.isabs(path) else path
    if os.path.exists(path):
        c = P.load_cluster_profile(path)
        if c.n_devices == n:
            return c, shown
        # re-scope a measured 8-GPU table to n devices
        table = tuple(e for e in c.bandwidth_table if e.group_size <= n)
        c = P.ClusterProfile(n, min(c.devices_per_node, n), c.device_flops,
                             c.device_memory_bytes, c.memory_reserve_fraction, table)
        c.validate()
        return c, shown + f" (rescoped to {n})"
    table = tuple(P.BandwidthEntry("intra_node", g, 700e9, 5e-6) for g in (2, 4, 8) if g <= n)
    c = P.ClusterProfile(n, min(n, 8), 1.2e15, 180_000_000_000, 0.1, table)
    c.validate()
    return c, "builtin placeholder (device_flops 1.2e15, busbw 7e11, reserve 0.1)"


def model_profile(cfg):
    """Planner ModelProfile: the profiler's activation-calibrated one when committed
    (profiles/b200_model_<name>.json, `profiler --model-out`), else the analytic one;
    both carry the embedding/head folded into the first/last layer
    (profiler.fold_embedding_head)."""
    from paper_2504_21411_b200.planner.profiles import load_model_profile
    from paper_2504_21411_b200.profiler import planned_profile
    path = os.path.join(ROOT, "profiles", f"b200_model_{cfg.name}.json")
    if os.path.exists(path):
        return load_model_profile(path)
    return planned_profile(cfg)


def training_config(cfg, n: int, global_batch: int):
    """TrainingConfig for the search: bytes per param/grad/optimizer state at the cost-model
    defaults and comm_overlap_fraction as measured by the profiler for this model at this
    world size (profiles/b200_training_<model>_n<N>.json, `profiler --overlap-out`); N
    beyond the largest measured world uses that world's fraction; none measured -> 0."""
    from paper_2504_21411_b200.planner.profiles import TrainingConfig, load_training_config
    best = None
    for k in (1, 2, 4, 8, 16):
        path = os.path.join(ROOT, "profiles", f"b200_training_{cfg.name}_n{k}.json")
        if k <= n and os.path.exists(path):
            best = path
    if n == 1 or best is None:
        return TrainingConfig(global_batch=global_batch), "comm_overlap_fraction 0 (no dp sync)" \
            if n == 1 else "comm_overlap_fraction 0 (not measured)"
    f = load_training_config(best).comm_overlap_fraction
    return (TrainingConfig(global_batch=global_batch, comm_overlap_fraction=f),
            f"comm_overlap_fraction {f:.4f} measured ({os.path.relpath(best, ROOT)})")


def plan_for(cfg, n: int, global_batch: int, cluster):
    from paper_2504_21411_b200.planner.profiles import TrainingConfig
    from paper_2504_21411_b200.planner.search import SearchConfig, optimize
    from paper_2504_21411_b200.runtime.config import get_hybrid_parallel_configs, profile_for
    training, _ = training_config(cfg, n, global_batch)
    mp = model_profile(cfg)
    plan = optimize(mp, cluster, training, SearchConfig())
    return plan, get_hybrid_parallel_configs(plan, cfg, model_profile=mp, cluster=cluster,
                                             training=training), training


def parse_pattern(text: str, n: int):
    """'tp8,dp8z3,tp4dp2sp,tp1dp8rc' -> [ParallelStrategy] (tp*dp must equal n)."""
    import re
    from paper_2504_21411_b200.planner.strategy import ParallelStrategy
    out = []
    for tok in text.split(","):
        m = re.fullmatch(r"(?:tp(\d+))?(?:dp(\d+))?(?:z(\d))?(sp)?(rc)?", tok.strip())
        if not m:
            raise SystemExit(f"bad strategy token {tok!r}")
        tp = int(m.group(1) or (n // int(m.group(2)) if m.group(2) else 1))
        dp = int(m.group(2) or n // tp)
        out.append(ParallelStrategy(tp, dp, int(m.group(3) or 0), bool(m.group(4)),
                                    bool(m.group(5))))
    return out


def explicit_plan(cfg, n, global_batch, cluster, pattern, microbatch, pp=1):
    from paper_2504_21411_b200.planner.profiles import TrainingConfig
    from paper_2504_21411_b200.planner.search import make_plan
    from paper_2504_21411_b200.runtime.config import get_hybrid_parallel_configs, profile_for
    strats = parse_pattern(pattern, n // pp)
    layers = [strats[i % len(strats)] for i in range(cfg.n_layers)]
    training, _ = training_config(cfg, n, global_batch)
    mp = model_profile(cfg)
    plan = make_plan(mp, cluster, training, pp, microbatch, layers)
    # hand-written plans are validated like searched ones: over budget -> InvalidPlan
    return plan, get_hybrid_parallel_configs(plan, cfg, model_profile=mp, cluster=cluster,
                                             training=training), training


def describe(hc) -> str:
    kinds = []
    for s in hc.layer_strategies:
        k = f"tp{s.tp}dp{s.dp}z{s.zero_stage}" + ("sp" if s.sp else "") + ("rc" if s.recompute else "")
        if not kinds or kinds[-1][0] != k:
            kinds.append([k, 1])
        else:
            kinds[-1][1] += 1
    names = [k for k, c in kinds for _ in range(c)]
    for period in range(1, len(names) // 2 + 1):
        if len(names) % period == 0 and names == names[:period] * (len(names) // period) \
                and period > 1:
            layers = "(" + "+".join(names[:period]) + f")x{len(names) // period}"
            break
    else:
        layers = "+".join(f"{k}x{c}" for k, c in kinds)
    return f"pp{hc.pp} mb{hc.microbatch}x{hc.n_microbatches} [{layers}]"


def memory_breakdown(plan, model, cluster, training, peak_gb, persistent_bytes):
    """This rank's stage: the cost model's terms (costmodel.py:137-176) next to the
    runtime's persistent bytes (after construction, symmetric pools included) and peak."""
    from paper_2504_21411_b200.planner import costmodel
    cfg = model.cfg
    prof = model_profile(cfg)
    st = model.stage
    lo, hi = plan.stage_ranges[st]
    infl = costmodel.in_flight_microbatches(plan.pp, st, plan.n_microbatches)
    tot = {"param": 0.0, "grad": 0.0, "optimizer": 0.0, "activation": 0.0}
    for li in range(lo, hi):
        m = costmodel.layer_memory(prof.layers[li], plan.layer_strategies[li], plan.microbatch,
                                   prof.seq_len, infl, training)
        tot["param"] += m.param_bytes
        tot["grad"] += m.grad_bytes
        tot["optimizer"] += m.optimizer_bytes
        tot["activation"] += m.activation_bytes
    state = tot["param"] + tot["grad"] + tot["optimizer"]
    last = plan.layer_strategies[hi - 1]
    return {"stage": st, "pp": plan.pp, "microbatch": plan.microbatch, "in_flight": infl,
            "seq_len": prof.seq_len, "last_layer": last.to_dict(),
            "first_layer": plan.layer_strategies[lo].to_dict(),
            "model_state_gb": state / 1e9, "model_activation_gb":
            tot["activation"] / 1e9, "runtime_persistent_gb": persistent_bytes / 1e9,
            "runtime_peak_gb": peak_gb, "predicted_gb": plan.predicted_stage_peak_memory[st] / 1e9,
            "budget_gb": cluster.memory_budget_bytes() / 1e9,
            "peak_within_prediction": peak_gb * 1e9 <= plan.predicted_stage_peak_memory[st]}


def write_report(path, plan, model, cluster, training, tokens, rank):
    """One instrumented step (per-layer CUDA events + step marks) -> report.py bundle."""
    import torch
    from paper_2504_21411_b200.report import measured_report, report_to_csv
    from paper_2504_21411_b200.planner.serialize import dumps_canonical
    model.layer_events.clear()
    model.trace.clear()
    model.record_layers = model.record_trace = True
    torch.cuda.reset_peak_memory_stats()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    model.train_step(tokens)
    model.wait_optimizer()
    b.record()
    torch.cuda.synchronize()
    model.record_layers = model.record_trace = False
    marks = {kind: ev for kind, _, ev in model.trace}
    exposed = marks["dp_sync"].elapsed_time(marks["end"]) / 1e3 if "dp_sync" in marks else None
    peak = torch.cuda.max_memory_allocated() + model.symmetric_bytes()
    bundle = measured_report(plan, model_profile(model.cfg), cluster, training,
                             stage=model.stage, layer_times=model.layer_times(),
                             iteration_s=a.elapsed_time(b) / 1e3, dp_sync_exposed_s=exposed,
                             peak_memory_bytes=peak)
    out = f"{path}.rank{rank}" if rank else path
    if rank == 0 or model.topo.stage_group.index == 0:
        with open(out + ".json", "w") as fh:
            fh.write(dumps_canonical(bundle, sort_keys=False))
        with open(out + ".csv", "w") as fh:
            fh.write(report_to_csv(bundle))
    st = [r for r in bundle["stages"] if r["stage"] == model.stage][0]
    return {"file": out + ".json", "stage": model.stage,
            "stage_per_microbatch_error": st.get("relative_error"),
            "iteration_error": bundle["total"]["relative_error"],
            "max_abs_layer_error": bundle["total"]["max_abs_layer_error"],
            "layers_within_10pct": f"{bundle['total']['layers_within_10pct']}/"
                                   f"{bundle['total']['layers_measured']}"}


# ----------------------------------------------------------------------------- CPU arm

_REF_PLANNER = r"""
import hashlib, json, os, sys, time
import hybridplan
from hybridplan import profiles as P, search, pipesim
from hybridplan.serialize import dumps_canonical
args = json.loads(sys.argv[1])
assert os.path.realpath(hybridplan.__file__).startswith(os.path.realpath(args["ref_dir"]))
model = P.load_model_profile(args["model"])
cluster = P.load_cluster_profile(args["cluster"])
training = P.TrainingConfig(global_batch=args["global_batch"],
                            comm_overlap_fraction=args["overlap"])
out = {"hybridplan": os.path.dirname(hybridplan.__file__)}
for jobs in args["jobs"]:
    t0 = time.perf_counter()
    plan = search.optimize(model, cluster, training, search.SearchConfig(jobs=jobs))
    out[f"optimize_s_jobs{jobs}"] = time.perf_counter() - t0
text = dumps_canonical(plan.to_dict(), sort_keys=False)
out["plan_sha256"] = hashlib.sha256(text.encode()).hexdigest()
out["predicted_iteration_time"] = plan.predicted_iteration_time
t0 = time.perf_counter()
sim = pipesim.simulate(plan, model, cluster, training)
out["simulate_s"] = time.perf_counter() - t0
out["sim_makespan"] = sim.makespan
print(json.dumps(out))
"""


def reference_planner_timing(cfg, n: int, global_batch: int, cluster_path: str) -> dict:
    """the reference's own optimize() (ref search.py:663; --jobs pool at
    search.py:605-610) and simulate() (pipesim.py:132), run from the unmodified package
    installed in baseline/_ref, timed on this host's cores -- single-threaded and with
    jobs = cores -- on the exact committed B200 profile JSON, next to this repository's
    planner on the same inputs (the plans must be byte-identical)."""
    import hashlib
    import tempfile
    from paper_2504_21411_b200.planner import profiles as P
    from paper_2504_21411_b200.planner.search import SearchConfig, optimize
    from paper_2504_21411_b200.planner.serialize import dumps_canonical
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "hybridplan")):
        return {"unavailable": "baseline/_ref not installed (see DESIGN.md §6)"}
    model_path = os.path.join(ROOT, "profiles", f"b200_model_{cfg.name}.json")
    if not os.path.exists(model_path):
        return {"unavailable": f"no committed model profile for {cfg.name}"}
    cluster, shown = cluster_profile(n, cluster_path)
    cores = len(os.sched_getaffinity(0))
    with tempfile.TemporaryDirectory() as td:
        cpath = os.path.join(td, "cluster.json")
        P.save_profiles(cpath, cluster=cluster)
        training, tsrc = training_config(cfg, n, global_batch)
        arg = json.dumps({"ref_dir": ref_dir, "model": model_path, "cluster": cpath,
                          "global_batch": global_batch, "jobs": [1, cores],
                          "overlap": training.comm_overlap_fraction})
        r = subprocess.run([sys.executable, "-c", _REF_PLANNER, arg], cwd=ref_dir,
                           capture_output=True, text=True, timeout=600,
                           env={**os.environ, "PYTHONPATH": ref_dir})
    if r.returncode != 0:
        return {"unavailable": "reference planner failed: " + r.stderr.strip()[-300:]}
    ref = json.loads(r.stdout.strip().splitlines()[-1])
    mp = P.load_model_profile(model_path)
    t0 = time.perf_counter()
    plan = optimize(mp, cluster, training, SearchConfig())
    ours_s = time.perf_counter() - t0
    sha = hashlib.sha256(dumps_canonical(plan.to_dict(), sort_keys=False).encode()).hexdigest()
    return {"inputs": {"model": os.path.relpath(model_path, ROOT), "cluster": shown,
                       "n_devices": n, "global_batch": global_batch, "training": tsrc},
            "cores": cores, "reference": ref, "ours_optimize_s_jobs1": ours_s,
            "plans_byte_identical": sha == ref.get("plan_sha256")}




def cpu_reference(cfg, steps: int, warmup: int):
    """The CPU restatement (oracle/model_ref.py) on a bounded sample: one decoder layer
    + embedding + head at microbatch 1 x seq_len in fp32, extrapolated to the full model
    by the FLOP ratio.  Returns (tokens/s, seconds per sample, cores, sample text)."""
    import torch
    from oracle import model_ref
    from paper_2504_21411_b200.runtime.init import full_weights, synthetic_tokens
    cores = len(os.sched_getaffinity(0))
    torch.set_num_threads(cores)
    one = cfg.with_(n_layers=1)
    w = full_weights(one)
    tokens = synthetic_tokens(one, 1)
    times = []
    for i in range(max(warmup, 0) + max(steps, 1)):
        t0 = time.perf_counter()
        model_ref.loss_and_grads(one, w, tokens, dtype=torch.float32)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
    t1 = statistics.median(times)
    scale = cfg.train_flops_per_token() / one.train_flops_per_token()
    t_full = t1 * scale
    tok_s = cfg.seq_len / t_full
    sample = (f"{cfg.name}: 1 decoder layer + embed + head, microbatch 1 x {cfg.seq_len} tokens, "
              f"fp32 fwd+bwd (oracle/model_ref.py), {t1:.2f}s/sample, extrapolated x{scale:.2f} "
              f"by training FLOPs to {cfg.n_layers} layers")
    return tok_s, t1, cores, sample


# ----------------------------------------------------------------------------- main


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    from paper_2504_21411_b200.runtime.config import MODEL_PRESETS
    cfg = MODEL_PRESETS[args.model]
    n = world
    gb = args.seqs_per_gpu * n
    metric = f"{cfg.name} train tokens/s"

    if args.impl == "reference":
        if rank != 0:
            return 0
        steps, warm = max(1, min(args.steps, 3)), min(args.warmup, 3)  # ~5 s per CPU step
        tok_s, t1, cores, sample = cpu_reference(cfg, steps, warm)
        # the search at this run's N and at the north star's 8 B200s
        planner = {f"n{k}": reference_planner_timing(
            cfg, k, args.seqs_per_gpu * k,
            args.cluster_profile or default_cluster_profile(args.model))
            for k in sorted({args.gpus, 8})}
        line = {"metric": metric, "value": tok_s, "unit": "tokens/s", "n_gpus": args.gpus,
                "steps": steps, "warmup": warm, "ms_per_step": t1 * 1e3,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f32", "data": "synthetic tokens, random-init weights",
                "impl": "reference",
                "config": {"workload": f"{cfg.name} training step (CPU restatement sample)",
                           "seq_len": cfg.seq_len},
                "cpu_baseline": {"value": tok_s, "unit": "tokens/s", "cores": cores,
                                 "kind": "port", "sample": sample},
                "e2e": {"value": tok_s, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0},
                "planner_cpu": planner}
        print(json.dumps(line), flush=True)
        return 0

    import torch
    import torch.distributed as dist
    os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    from paper_2504_21411_b200 import kernels as K
    from paper_2504_21411_b200.runtime.engine import construct_hybrid_parallel_model
    from paper_2504_21411_b200.runtime.init import synthetic_tokens

    cluster, cluster_src = cluster_profile(
        n, args.cluster_profile or default_cluster_profile(args.model))
    if args.layer_pattern:
        plan, hc, training = explicit_plan(cfg, n, gb, cluster, args.layer_pattern,
                                           args.microbatch or max(n // args.pp, 1), args.pp)
    else:
        plan, hc, training = plan_for(cfg, n, gb, cluster)
    if args.sp_mode != "megatron":
        import dataclasses
        hc = dataclasses.replace(hc, sp_mode=args.sp_mode)
    if args.plan_out and rank == 0:
        from paper_2504_21411_b200.planner.serialize import dumps_canonical
        with open(args.plan_out, "w") as fh:
            fh.write(dumps_canonical(plan.to_dict(), sort_keys=False))
    model = construct_hybrid_parallel_model(cfg, hc, training=training, dtype=torch.bfloat16,
                                            init="fast")
    torch.cuda.synchronize()
    persistent_bytes = torch.cuda.memory_allocated() + model.symmetric_bytes()
    tokens_host = synthetic_tokens(cfg, gb).pin_memory()
    tokens_dev = tokens_host.to("cuda")
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    for _ in range(args.warmup):
        model.train_step(tokens_dev)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()

    # ---- device-resident timed region (launch count only: a host-side counter)
    stats = K.start_stats(time_gemm=False)
    with ClockSampler(local_rank) as clocks:
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record()
        for _ in range(args.steps):
            model.train_step(tokens_dev)
        model.wait_optimizer()  # the last step's AdamW runs on a side stream
        end.record()
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
    K.stop_stats()
    ms = max_over_ranks(start.elapsed_time(end) / args.steps)
    tokens_per_step = gb * cfg.seq_len
    value = tokens_per_step / (ms / 1e3)
    launches = stats.launches // args.steps * args.steps

    # ---- roofline pass (separate, so the per-GEMM CUDA events stay out of `value`): every
    # GEMM launch of a few more steps bracketed by events on its launching stream
    rsteps = min(args.steps, 3)
    stats = K.start_stats(time_gemm=True)
    r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    r0.record()
    for _ in range(rsteps):
        model.train_step(tokens_dev)
    model.wait_optimizer()
    r1.record()
    torch.cuda.synchronize()
    K.stop_stats()
    gemm = stats.gemm_summary()
    roof_ms = r0.elapsed_time(r1)

    # ---- end-to-end through the public API with host buffers
    barrier()
    torch.cuda.synchronize()
    e0 = time.perf_counter()
    st_e, en_e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st_e.record()
    for _ in range(args.steps):
        loss = model.train_step(tokens_host)
        loss_val = float(loss.item())
    model.wait_optimizer()
    en_e.record()
    torch.cuda.synchronize()
    barrier()
    e_ms = max_over_ranks(st_e.elapsed_time(en_e) / args.steps)
    e2e = tokens_per_step / (e_ms / 1e3)

    peaks, peak_src = measured_peaks()
    # DRAM traffic of the dominant kernel from the committed ncu --set full capture
    # (tools/gemm_one.py under ncu: the gate|up GEMM + SwiGLU epilogue, the step's largest
    # launch; profiles/r02/ncu/gemm_gateup_summary.json)
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "ncu", "gemm_gateup_summary.json")) as fh:
            cap = json.load(fh)
        rd = float(cap["dram__bytes_read.sum"].split()[0]) * 1e6
        wr = float(cap["dram__bytes_write.sum"].split()[0]) * 1e6
        traffic = {"bytes_per_launch": rd + wr,
                   "shape": "8192x22016x4096 gate|up fwd + SwiGLU epilogue (mb2)",
                   "algorithmic_bytes": 2 * (8192 * 4096 + 22016 * 4096 + 8192 * 22016
                                             + 8192 * 11008),
                   "source": "profiles/r02/ncu/gemm_gateup_summary.json (ncu --set full)"}
    except (OSError, KeyError, ValueError, IndexError):
        pass
    flops_tok = cfg.train_flops_per_token()
    mfu = value * flops_tok / (n * PEAK_BF16_DENSE)
    peak_tf = peaks.get("bf16_tflops_sustained", 1424.5)
    clk = clocks.summary()
    # caching-allocator peak + the symmetric (NVLink) dp pools and tp peer buffers, which
    # live outside it
    mem = (torch.cuda.max_memory_allocated() + model.symmetric_bytes()) / 1e9
    alloc_retries = torch.cuda.memory_stats().get("num_alloc_retries", 0)
    line = {
        "metric": metric, "value": value, "unit": "tokens/s", "n_gpus": n,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic tokens (seeded randint), random-init weights",
        "config": {"workload": f"{cfg.name} training step (fwd+bwd+AdamW)", "model": cfg.name,
                   "global_batch": gb, "seq_len": cfg.seq_len,
                   "parallelism": describe(hc) + ("" if hc.sp_mode == "megatron"
                                                  else f" sp_mode={hc.sp_mode}"),
                   "l2": "working set (weights/activations) >> 126 MB L2; no flush"},
        "mfu": mfu, "mfu_basis": "2.25 PFLOP/s dense bf16 per GPU; attention counted "
                                 "non-causal (12*L*h*s per token, the cost model's "
                                 "flops_per_token_sq = 4h convention)",
        "mfu_causal": value * cfg.train_flops_per_token_causal() / (n * PEAK_BF16_DENSE),
        "flops_per_token": flops_tok,
        "predicted_iteration_time_s": plan.predicted_iteration_time,
        "measured_iteration_time_s": ms / 1e3,
        "prediction_error": (ms / 1e3 - plan.predicted_iteration_time) / plan.predicted_iteration_time,
        "cluster_profile": cluster_src,
        "training_config": training_config(cfg, n, gb)[1],
        "model_profile": ("profiles/b200_model_%s.json (activation-calibrated)" % cfg.name
                          if os.path.exists(os.path.join(ROOT, "profiles",
                                                         "b200_model_%s.json" % cfg.name))
                          else "analytic (profiler.planned_profile: profile_for + embedding/head fold)"),
        "roofline": {"bound": "tensor", "kernel": "galv tcgen05 GEMM (all shapes of the step)",
                     "achieved": gemm["tflops"], "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": gemm["tflops"] / peak_tf if peak_tf else None,
                     "traffic": traffic["bytes_per_launch"] if traffic else None,
                     "traffic_detail": traffic, "peak_source": f"{peak_src} bf16_tflops_sustained",
                     "gemm_share_of_step": gemm["ms"] / roof_ms,
                     "measured_over": f"{rsteps} extra steps with per-GEMM CUDA events "
                                      "(not inside the `value` region)",
                     "gemm_launches": gemm["launches"]},
        "gpu_launches": launches,
        "e2e": {"value": e2e, "unit": "tokens/s",
                "h2d_bytes_per_step": tokens_host.numel() * tokens_host.element_size(),
                "d2h_bytes_per_step": 4},
        "clocks": clk, "loss": loss_val, "peak_mem_gb": mem, "alloc_retries": alloc_retries,
        "dp_collectives": ({"impl": "nvlink", "pools": len(model.dp_pools),
                            "multicast": all(bool(p.mc) for p in model.dp_pools)}
                           if model.dp_pools else {"impl": "nccl" if n > 1 else "none"}),
        "predicted_peak_mem_gb": max(plan.predicted_stage_peak_memory) / 1e9,
        "memory": memory_breakdown(plan, model, cluster, training, mem, persistent_bytes),
    }
    if args.report_out:
        line["report"] = write_report(args.report_out, plan, model, cluster, training,
                                      tokens_dev, rank)
    if args.trace_out:
        model.record_trace = True
        model.trace.clear()
        model.train_step(tokens_dev)
        model.record_trace = False
        measured = model.measured_trace()
        from paper_2504_21411_b200.planner.pipesim import simulate, trace_to_jsonl, SimResult
        from paper_2504_21411_b200.runtime.config import profile_for
        sim = simulate(plan, model_profile(cfg), cluster, training)
        def per_kind(events):
            acc = {}
            for e in events:
                acc.setdefault(e.kind, []).append(e.duration)
            return {k: {"n": len(v), "mean_s": sum(v) / len(v)} for k, v in acc.items()}
        diff = {"measured": per_kind(measured),
                "simulated": per_kind([e for e in sim.trace if e.device_stage == model.stage]),
                "measured_makespan_s": sum(e.duration for e in measured),
                "simulated_makespan_s": sim.makespan}
        if rank == 0 or model.stage > 0:
            with open(f"{args.trace_out}.rank{rank}.jsonl", "w") as fh:
                fh.write(trace_to_jsonl(SimResult(0.0, (), tuple(measured), 0.0)))
            with open(f"{args.trace_out}.rank{rank}.diff.json", "w") as fh:
                json.dump(diff, fh, indent=1)
        line["trace_diff"] = diff
    if rank == 0 and n == 1 and not args.no_cpu_baseline:
        tok_s, t1, cores, sample = cpu_reference(cfg, 1, 0)
        line["cpu_baseline"] = {"value": tok_s, "unit": "tokens/s", "cores": cores,
                                "kind": "port", "sample": sample}
        # the reference planner itself (baseline/_ref) on the committed profiles, N=8
        line["planner_cpu"] = {"n8": reference_planner_timing(
            cfg, 8, args.seqs_per_gpu * 8,
            args.cluster_profile or default_cluster_profile(args.model))}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
