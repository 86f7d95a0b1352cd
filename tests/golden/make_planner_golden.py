"""Generate planner golden vectors by running the REFERENCE planner.

Run in the build container (where /root/reference exists):

    python tests/golden/make_planner_golden.py               # random + BASELINE instances
    python tests/golden/make_planner_golden.py --committed   # the committed B200 profiles

It imports the reference ``hybridplan`` read-only from /root/reference/pkg/src
(never copied into this repo) and writes ``planner_golden.jsonl``: one line
per instance with the canonical input profile documents and the reference's
outputs (Plan JSON bytes from ``optimize``, ``optimize_with_report`` flags,
``simulate`` makespan/peaks/bubble and a SHA-256 of its JSONL trace, and the
``build_report`` CSV digest).  ``tests/test_planner_parity.py`` replays every
line through ``paper_2504_21411_b200.planner`` and requires byte equality.
"""

from __future__ import annotations

import hashlib
import json
import math
import random
import sys
from pathlib import Path

REF = "/root/reference/pkg/src"
OUT = Path(__file__).with_name("planner_golden.jsonl")


def _instances(ref, seed: int, count: int):
    """Seeded random small instances, half of them with a binding memory budget."""
    P = ref.profiles
    rng = random.Random(seed)
    made = 0
    while made < count:
        n = rng.choice([1, 2, 4, 8])
        per_node = rng.choice([d for d in (1, 2, 4, 8) if d <= n])
        table = []
        g = 2
        ibw, ilat = 10 ** rng.uniform(10.5, 11.7), rng.choice([0.0, 1e-7, 2e-6])
        xbw, xlat = 10 ** rng.uniform(9.5, 10.5), rng.choice([0.0, 1e-6, 5e-6])
        while g <= per_node:
            table.append(P.BandwidthEntry("intra_node", g, ibw * (1.0 - 0.05 * math.log2(g)), ilat))
            g *= 2
        g = 2
        while g <= n:
            table.append(P.BandwidthEntry("inter_node", g, xbw, xlat))
            g *= 2
        layers = []
        n_layers = rng.randint(1, 6)
        hidden = rng.choice([32, 64, 128, 256])
        seq = rng.choice([16, 32, 64, 128])
        uniform = rng.random() < 0.4
        for _ in range(n_layers):
            if uniform and layers:
                layers.append(layers[0])
                continue
            params = rng.uniform(1e4, 4e6)
            shard = rng.uniform(4, 40) * hidden
            repl = rng.uniform(2, 16) * hidden
            layers.append(P.LayerProfile(params, 2.0 * params, rng.uniform(0, 8) * hidden,
                                         shard, repl, min(rng.uniform(0.5, 2.0) * hidden,
                                                          shard + repl)))
        model = P.ModelProfile(n_layers, hidden, seq, tuple(layers))
        training = P.TrainingConfig(global_batch=max(n, 1) * rng.choice([1, 2, 4, 8]),
                                    comm_overlap_fraction=rng.choice([0.0, 0.0, 0.25, 0.5]))
        memory = 1 << 50
        cluster = P.ClusterProfile(n, per_node, 10 ** rng.uniform(9, 12), memory,
                                   rng.choice([0.0, 0.05]), tuple(table))
        if rng.random() < 0.5:
            # squeeze memory near the unconstrained plan's peak to make it bind
            try:
                free = ref.search.optimize(model, cluster, training)
            except ref.errors.PlannerError:
                continue
            peak = max(free.predicted_stage_peak_memory)
            memory = max(int(peak * rng.uniform(0.2, 1.1)), 1024)
            cluster = P.ClusterProfile(n, per_node, cluster.device_flops, memory,
                                       cluster.memory_reserve_fraction, tuple(table))
        yield cluster, model, training, {
            "transitions": rng.random() < 0.8, "memory_buckets": rng.choice([64, 256, 1024])}
        made += 1


def _b200_configs(ref):
    """BASELINE.json configs with a flat placeholder B200 profile."""
    P = ref.profiles
    out = []
    for n in (1, 2, 4, 8):
        table = tuple(P.BandwidthEntry("intra_node", g, 700e9, 5e-6) for g in (2, 4, 8) if g <= n)
        cl = P.ClusterProfile(n, n, 1424.5e12, 180_000_000_000, 0.0, table)
        for name, L, h, s, gbs in (("gpt2m", 24, 1024, 1024, 16), ("gpt1.3b", 24, 2048, 2048, 8),
                                   ("tiny", 4, 512, 256, 8)):
            out.append((name, cl, P.synth_transformer_profile(L, h, s),
                        P.TrainingConfig(global_batch=gbs * n)))
    return out


# committed B200 profiles (profiles/*.json) x the headline device counts: the exact plan
# inputs bench.py searches on, pinned to the reference's choice
COMMITTED = (("llama2-7b", "b200_cluster.json", 8, (1, 2, 4, 8)),
             ("llama2-13b", "b200_cluster_llama13b_180g.json", 2, (4, 8)),
             ("gpt2-medium", "b200_cluster_gpt2m.json", 16, (1, 2, 4, 8)),
             ("gpt-1.3b", "b200_cluster.json", 16, (4, 8)))
OUT_B200 = Path(__file__).with_name("planner_golden_b200.jsonl")


def _committed(ref):
    """(tag, cluster, model, training) for every COMMITTED profile pair, the cluster
    re-scoped to n devices exactly as bench.cluster_profile does."""
    P = ref.profiles
    prof = Path(__file__).resolve().parents[2] / "profiles"
    for name, cl_file, per_gpu, ns in COMMITTED:
        model = P.load_model_profile(str(prof / f"b200_model_{name}.json"))
        base = P.load_cluster_profile(str(prof / cl_file))
        for n in ns:
            table = tuple(e for e in base.bandwidth_table if e.group_size <= n)
            cl = P.ClusterProfile(n, min(base.devices_per_node, n), base.device_flops,
                                  base.device_memory_bytes, base.memory_reserve_fraction, table)
            # bench.training_config: the measured comm_overlap_fraction of the largest
            # measured world <= n (profiles/b200_training_<model>_n<k>.json), else 0
            overlap = 0.0
            for k in (2, 4, 8, 16):
                tpath = prof / f"b200_training_{name}_n{k}.json"
                if n > 1 and k <= n and tpath.exists():
                    overlap = P.load_training_config(str(tpath)).comm_overlap_fraction
            yield (f"committed-{name}-n{n}", cl, model,
                   P.TrainingConfig(global_batch=per_gpu * n, comm_overlap_fraction=overlap))


def main_committed(ref) -> None:
    from hybridplan import pipesim as refsim
    with open(OUT_B200, "w") as fh:
        for tag, cl, mo, tr in _committed(ref):
            plan = ref.search.optimize(mo, cl, tr)
            sim = refsim.simulate(plan, mo, cl, tr)
            doc = {"tag": tag, "cluster": ref.profiles.cluster_to_dict(cl),
                   "model": ref.profiles.model_to_dict(mo),
                   "training": ref.profiles.training_to_dict(tr),
                   "plan": ref.serialize.dumps_canonical(plan.to_dict(), sort_keys=False),
                   "sim": {"makespan": sim.makespan, "peaks": list(sim.stage_peak_memory),
                           "trace_sha256": hashlib.sha256(
                               refsim.trace_to_jsonl(sim).encode()).hexdigest()}}
            fh.write(json.dumps(doc, sort_keys=True) + "\n")
            print(tag, plan.pp, plan.microbatch, plan.predicted_iteration_time)
    print(f"wrote {OUT_B200}")


def main() -> None:
    sys.path.insert(0, REF)
    if "--committed" in sys.argv:
        import hybridplan as ref  # noqa: E402
        import hybridplan.profiles  # noqa: F401,E402
        import hybridplan.search  # noqa: F401,E402
        main_committed(ref)
        return
    import hybridplan as ref  # noqa: E402
    from hybridplan import cli as refcli, pipesim as refsim  # noqa: E402
    import hybridplan.profiles  # noqa: F401,E402
    import hybridplan.search  # noqa: F401,E402

    lines = []

    def record(tag, cluster, model, training, knobs):
        doc = {"tag": tag,
               "cluster": ref.profiles.cluster_to_dict(cluster),
               "model": ref.profiles.model_to_dict(model),
               "training": ref.profiles.training_to_dict(training),
               "knobs": knobs}
        cfg = ref.search.SearchConfig(transitions=knobs["transitions"],
                                      memory_buckets=knobs["memory_buckets"])
        try:
            rep = ref.search.optimize_with_report(model, cluster, training, cfg)
        except ref.errors.NoFeasiblePlan as exc:
            doc["infeasible"] = {"stage_index": exc.stage_index,
                                 "min_achievable_bytes": exc.min_achievable_bytes,
                                 "budget_bytes": exc.budget_bytes, "message": str(exc)}
            lines.append(doc)
            return
        plan = rep.plan
        doc["plan"] = ref.serialize.dumps_canonical(plan.to_dict(), sort_keys=False)
        doc["memory_binding"] = rep.memory_binding
        sim = refsim.simulate(plan, model, cluster, training, transitions=knobs["transitions"])
        doc["sim"] = {"makespan": sim.makespan, "peaks": list(sim.stage_peak_memory),
                      "bubble": sim.bubble_fraction, "n_events": len(sim.trace),
                      "trace_sha256": hashlib.sha256(
                          refsim.trace_to_jsonl(sim).encode()).hexdigest()}
        bundle = refcli.build_report(plan, model, cluster, training,
                                     transitions=knobs["transitions"])
        doc["report_sha256"] = hashlib.sha256(
            (ref.serialize.dumps_canonical(bundle, sort_keys=False)
             + refcli.report_to_csv(bundle)).encode()).hexdigest()
        lines.append(doc)

    for i, (cl, mo, tr, knobs) in enumerate(_instances(ref, 20261018, 240)):
        record(f"random{i}", cl, mo, tr, knobs)
    for name, cl, mo, tr in _b200_configs(ref):
        record(f"b200-{name}-n{cl.n_devices}", cl, mo, tr,
               {"transitions": True, "memory_buckets": 1024})
    with open(OUT, "w") as fh:
        for doc in lines:
            fh.write(json.dumps(doc, sort_keys=True) + "\n")
    print(f"wrote {len(lines)} instances to {OUT}")


if __name__ == "__main__":
    main()
