"""Measured-vs-predicted report in the reference's report bundle format.

``build_report`` (reference cli.py:213-292, restated in planner/cli.py) gives the cost
model's per-layer / per-stage / total rows for a Plan; ``measured_report`` adds, for this
rank's pipeline stage, the same rows measured on the GPU from one instrumented training
step (engine.record_layers: CUDA events around every layer forward / backward, every
layout transition, the embedding and the head, on the compute stream):

* layer: ``measured_fwd`` / ``measured_bwd`` (recompute replay, tp collectives and
  ZeRO-3 gathers included, as the model's fwd + bwd + recompute_extra + tp_comm +
  zero3_param_gather), ``measured_transition`` (fwd + bwd reshard into the layer), the
  head / embedding time on the layers they are folded into (profiler.fold_embedding_head),
  ``measured_time_total`` and ``relative_error`` against the model's ``time_total``;
* stage: ``measured_per_microbatch_time`` (sum of its layers' measured totals) against
  ``per_microbatch_time``, the measured step-end dp-sync exposure against
  ``dp_sync_time``, the measured peak memory against ``peak_memory_bytes``;
* total: measured iteration time against ``predicted_iteration_time`` and the simulated
  1F1B makespan (pipesim.compare_with_analytic, reference pipesim.py:241).

``report_to_csv`` writes the reference CSV columns plus the measured ones.
"""

from __future__ import annotations

from collections import defaultdict

from .planner import cli
from .planner.serialize import format_float


def _mean(v):
    return sum(v) / len(v) if v else 0.0


def measured_report(plan, model, cluster, training, *, stage: int, layer_times: list,
                    iteration_s: float, dp_sync_exposed_s: float | None = None,
                    peak_memory_bytes: int | None = None, transitions: bool = True) -> dict:
    bundle = cli.build_report(plan, model, cluster, training, transitions=transitions)
    acc = defaultdict(list)
    for kind, li, mb, sec in layer_times:
        acc[(kind, li, mb)].append(sec)
    per = defaultdict(lambda: defaultdict(list))  # layer -> kind -> [seconds per microbatch]
    for (kind, li, mb), secs in acc.items():
        per[li][kind].append(sum(secs))
    lo, hi = plan.stage_ranges[stage]
    stage_total = 0.0
    for row in bundle["layers"]:
        li = row["layer"]
        if not lo <= li < hi:
            continue
        k = per.get(li, {})
        fwd, bwd = _mean(k.get("fwd", [])), _mean(k.get("bwd", []))
        trans = _mean(k.get("transition_fwd", [])) + _mean(k.get("transition_bwd", []))
        extra = (_mean(k.get("head", [])) + _mean(k.get("embed_fwd", []))
                 + _mean(k.get("embed_bwd", [])))
        total = fwd + bwd + trans + extra
        stage_total += total
        row.update({"measured_fwd": fwd, "measured_bwd": bwd, "measured_transition": trans,
                    "measured_embedding_head": extra, "measured_time_total": total,
                    "relative_error": (total - row["time_total"]) / row["time_total"]
                    if row["time_total"] else None})
    for li, tr in transition_traffic(plan, model, hidden=model.hidden_size).items():
        bundle["layers"][li].update(tr)
    for row in bundle["stages"]:
        if row["stage"] != stage:
            continue
        pred = row["per_microbatch_time"]
        row.update({"measured_per_microbatch_time": stage_total,
                    "relative_error": (stage_total - pred) / pred if pred else None,
                    "measured_dp_sync_exposed": dp_sync_exposed_s,
                    "measured_peak_memory_bytes": peak_memory_bytes,
                    "peak_within_prediction": (peak_memory_bytes <= row["peak_memory_bytes"]
                                               if peak_memory_bytes is not None else None)})
    tot = bundle["total"]
    tot.update({"measured_iteration_time": iteration_s,
                "relative_error": (iteration_s - tot["predicted_iteration_time"])
                / tot["predicted_iteration_time"], "measured_stage": stage})
    errs = [abs(r["relative_error"]) for r in bundle["layers"]
            if r.get("relative_error") is not None]
    tot["max_abs_layer_error"] = max(errs) if errs else None
    tot["layers_within_10pct"] = sum(e <= 0.10 for e in errs)
    tot["layers_measured"] = len(errs)
    return bundle


def transition_traffic(plan, model, *, hidden: int, act_bytes: int = 2) -> dict:
    """Per layer with a layout change: the bytes the busiest rank sends in the runtime's
    reshard (runtime/reshard.plan_transition: rows a rank already holds never move) next
    to the volume the cost model charges (transition_time = all-gather of microbatch*s*
    boundary bytes over the stage group, costmodel.py:179-196, i.e. (g-1)/g of it per rank
    on the ring)."""
    from .runtime.reshard import Layout, plan_transition
    out = {}
    T = plan.microbatch * model.seq_len
    for i, (lo, hi) in enumerate(plan.stage_ranges):
        for li in range(lo + 1, hi):
            a, b = plan.layer_strategies[li - 1], plan.layer_strategies[li]
            if a.same_layout(b):
                continue
            src, dst = Layout.of(a), Layout.of(b)
            tp = plan_transition(src, dst, T)
            g = src.tp * src.dp
            sent = [sum(max(h - l, 0) for j, (l, h) in enumerate(tp.send_rows[r]) if j != r)
                    for r in range(g)]
            bound = (g - 1) / g * T * model.layers[li].boundary_bytes_per_token
            out[li] = {"reshard_bytes_max_rank": max(sent) * hidden * act_bytes,
                       "model_allgather_bytes_per_rank": bound}
    return out


COLUMNS = cli.CSV_COLUMNS + ["measured_time_total", "relative_error"]


def _cell(v) -> str:
    if v is None:
        return ""
    if isinstance(v, bool):
        return "true" if v else "false"
    if isinstance(v, float):
        return format_float(v)
    return str(v)


def report_to_csv(bundle: dict) -> str:
    """The reference report CSV (cli.report_to_csv columns) + measured total and error."""
    base = cli.report_to_csv(bundle).splitlines()
    rows = [",".join(COLUMNS)]
    extra = ([(r.get("measured_time_total"), r.get("relative_error")) for r in bundle["layers"]]
             + [(r.get("measured_per_microbatch_time"), r.get("relative_error"))
                for r in bundle["stages"]]
             + [(bundle["total"].get("measured_iteration_time"),
                 bundle["total"].get("relative_error"))])
    for line, (m, e) in zip(base[1:], extra):
        rows.append(line + "," + _cell(m) + "," + _cell(e))
    return "\n".join(rows) + "\n"
