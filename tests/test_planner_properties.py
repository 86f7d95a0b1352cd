"""Planner known-answer and property tests (the reference's acceptance criteria,
re-derived: reference tests/test_acceptance.py:38-270)."""

import random
from fractions import Fraction

import pytest

from paper_2504_21411_b200.planner import (BandwidthEntry, ClusterProfile, LayerProfile,
                                           ModelProfile, ParallelStrategy, SearchConfig,
                                           StrategyConstraints, TrainingConfig, cli,
                                           costmodel, enumerate_strategies, make_plan,
                                           optimize, optimize_with_report, simulate,
                                           synth_transformer_profile, validate_plan)
from paper_2504_21411_b200.planner.collectives import (all_gather_time, all_reduce_time,
                                                       comm_group, p2p_time,
                                                       reduce_scatter_time)
from paper_2504_21411_b200.planner.errors import NoFeasiblePlan, ValidationError
from paper_2504_21411_b200.planner.search import brute_force_optimize


def cluster(n, per_node=None, *, flops=1e12, mem=32 << 30, intra=(300e9, 1e-6),
            inter=(25e9, 5e-6)):
    per_node = per_node or n
    table = [BandwidthEntry("intra_node", g, *intra) for g in (2, 4, 8, 16) if g <= per_node]
    table += [BandwidthEntry("inter_node", g, *inter) for g in (2, 4, 8, 16)
              if g <= n and per_node < n]
    c = ClusterProfile(n, per_node, flops, mem, 0.0, tuple(table))
    c.validate()
    return c


def test_strategy_space_counts_and_order():
    c = cluster(8)
    for d, count in ((1, 2), (2, 12), (4, 28), (8, 44)):
        got = enumerate_strategies(d, c)
        ref = [(tp, d // tp, z, sp, rc)
               for tp in (1, 2, 4, 8) if tp <= d
               for z in (0, 1, 2, 3) if z == 0 or d // tp > 1
               for sp in (False, True) if not (sp and tp == 1)
               for rc in (False, True)]
        assert len(got) == count
        assert [(s.tp, s.dp, s.zero_stage, s.sp, s.recompute) for s in got] == ref
    forced = enumerate_strategies(8, c, StrategyConstraints(force_recompute=True))
    assert len(forced) == 22 and all(s.recompute for s in forced)


def test_strategy_invariants():
    with pytest.raises(ValidationError):
        ParallelStrategy(1, 2, 0, True, False).validate()
    with pytest.raises(ValidationError):
        ParallelStrategy(2, 1, 1, False, False).validate()
    with pytest.raises(ValidationError):
        ParallelStrategy(2, 2, 0, False, False).validate(8)
    s = ParallelStrategy(2, 4, 3, True, True)
    assert ParallelStrategy.from_dict(s.to_dict()) == s
    assert s.same_layout(ParallelStrategy(2, 4, 0, True, False))


def test_collective_worked_numbers():
    c = cluster(8, intra=(1e11, 0.0))
    g4 = comm_group(c, 4)
    assert all_gather_time(g4, 1e9, c) == pytest.approx(0.0075)
    assert all_reduce_time(g4, 1e9, c) == pytest.approx(0.015)
    assert all_reduce_time(comm_group(c, 1), 1e9, c) == 0.0
    c2 = cluster(16, 8, inter=(2.5e10, 5e-6))
    assert all_gather_time(comm_group(c2, 16), 2e8, c2) == pytest.approx(
        15 * 5e-6 + (15 / 16) * 2e8 / 2.5e10)
    assert p2p_time(1e8, cluster(2, intra=(1e10, 0.0)), "intra_node") == pytest.approx(0.01)
    for g in (2, 4, 8):
        for v in (0.0, 1.0, 1e6, 1e9):
            grp = comm_group(c, g)
            assert all_reduce_time(grp, v, c) == reduce_scatter_time(grp, v, c) + \
                all_gather_time(grp, v, c)


def test_costmodel_worked_numbers():
    layer = synth_transformer_profile(1, 2, 8).layers[0]
    assert layer.param_count == 74
    c = cluster(1, flops=1e6)
    t = costmodel.layer_time(layer, ParallelStrategy(1, 1, 0, False, False), 4, 8, 2, c,
                             TrainingConfig(global_batch=8))
    assert t.fwd_compute == pytest.approx(6.784e-3)
    assert t.bwd_compute == pytest.approx(1.3568e-2)
    big = synth_transformer_profile(1, 1024, 1024).layers[0]
    tr = TrainingConfig(global_batch=8)
    m = costmodel.layer_memory(big, ParallelStrategy(2, 2, 0, False, False), 2, 1024, 1, tr)
    assert (m.param_bytes, m.optimizer_bytes) == (12_596_224.0, 75_577_344.0)
    assert costmodel.layer_memory(big, ParallelStrategy(2, 2, 1, False, False), 2, 1024, 1,
                                  tr).optimizer_bytes == 37_788_672.0
    assert costmodel.layer_memory(big, ParallelStrategy(2, 1, 0, True, False), 2, 1024, 1,
                                  tr).activation_bytes == 35_651_584.0
    assert costmodel.layer_memory(big, ParallelStrategy(2, 1, 0, True, True), 2, 1024, 1,
                                  tr).activation_bytes == 4_194_304.0


def _rand_instance(rng):
    n = rng.choice([2, 4, 8])
    per_node = rng.choice([d for d in (1, 2, 4, 8) if d <= n])
    c = cluster(n, per_node, flops=10 ** rng.uniform(9, 11), mem=1 << 60,
                intra=(10 ** rng.uniform(10.5, 11.5), rng.choice([0.0, 1e-6])),
                inter=(10 ** rng.uniform(9.5, 10.5), rng.choice([0.0, 5e-6])))
    hidden = rng.choice([32, 64])
    layers = []
    for _ in range(rng.randint(1, 3)):
        p = rng.uniform(1e4, 2e6)
        sh, rp = rng.uniform(4, 40) * hidden, rng.uniform(2, 16) * hidden
        layers.append(LayerProfile(p, 2 * p, rng.uniform(0, 8) * hidden, sh, rp,
                                   min(rng.uniform(0.5, 2) * hidden, sh + rp)))
    model = ModelProfile(len(layers), hidden, rng.choice([16, 32]), tuple(layers))
    return c, model, TrainingConfig(global_batch=n * rng.choice([1, 2]))


def test_search_equals_bruteforce_oracle_when_memory_is_free():
    rng = random.Random(7)
    for _ in range(25):
        c, model, tr = _rand_instance(rng)
        a = optimize(model, c, tr).predicted_iteration_time
        b = brute_force_optimize(model, c, tr).predicted_iteration_time
        assert abs(a - b) <= 1e-9 * b


def test_balanced_pipeline_simulation_is_exact():
    for pp in (1, 2, 4):
        for m in (1, 2, 4, 8):
            layer = LayerProfile(1024.0, 2.0 ** 20 / 8, 0.0, 64.0, 0.0, 0.0)
            model = ModelProfile(pp, 8, 8, (layer,) * pp)
            c = cluster(pp, flops=2.0 ** 20, intra=(300e9, 0.0), inter=(25e9, 0.0)) \
                if pp > 1 else ClusterProfile(1, 1, 2.0 ** 20, 1 << 30, 0.0, ())
            plan = make_plan(model, c, TrainingConfig(global_batch=m), pp, 1,
                             [ParallelStrategy(1, 1, 0, False, False)] * pp)
            res = simulate(plan, model, c, TrainingConfig(global_batch=m))
            assert Fraction(res.makespan) == (m + pp - 1) * Fraction(
                plan.cost_breakdown[0].per_microbatch_time)


def test_recompute_only_when_memory_binds():
    model = synth_transformer_profile(2, 64, 64)
    tr = TrainingConfig(global_batch=8)
    roomy = cluster(1, flops=1e9)
    plan = optimize(model, roomy, tr)
    assert not any(s.recompute for s in plan.layer_strategies)
    full = sum(costmodel.layer_memory(l, ParallelStrategy(1, 1, 0, False, False), 1, 64, 1,
                                      tr).total_int() for l in model.layers)
    tight = ClusterProfile(1, 1, 1e9, full - 1, 0.0, ())
    rep = optimize_with_report(model, tight, tr)
    assert any(s.recompute for s in rep.plan.layer_strategies) and rep.memory_binding
    assert validate_plan(rep.plan, model, tight, tr) == []


def test_cli_exit_codes(tmp_path):
    assert cli.main(["synth-profile", "--model", "--layers", "4", "--seq", "8",
                     "-o", str(tmp_path / "m.json")]) == 2
    assert cli.main(["synth-profile", "--model", "--layers", "1", "--hidden", "8", "--seq", "8",
                     "-o", str(tmp_path / "nodir" / "m.json")]) == 3
    assert cli.main(["bogus"]) == 2
    p = str(tmp_path / "p.json")
    assert cli.main(["synth-profile", "--model", "--layers", "2", "--hidden", "64", "--seq",
                     "32", "--cluster", "--devices", "2", "--training", "--global-batch", "8",
                     "-o", p]) == 0
    plan = str(tmp_path / "plan.json")
    assert cli.main(["search", "--cluster", p, "--model", p, "--training", p, "-o", plan]) == 0
    assert cli.main(["validate", "--cluster", p, "--model", p, "--training", p,
                     "--plan", plan]) == 0
    assert cli.main(["simulate", "--cluster", p, "--model", p, "--training", p, "--plan", plan,
                     "-o", str(tmp_path / "sim.json"), "--trace",
                     str(tmp_path / "t.jsonl")]) == 0
    assert cli.main(["report", "--cluster", p, "--model", p, "--training", p, "--plan", plan,
                     "-o", str(tmp_path / "rep")]) == 0
    import json
    pp = json.loads(open(plan).read())["pp"]
    assert (tmp_path / "rep.csv").read_text().count("\n") == 1 + 2 + pp + 1
