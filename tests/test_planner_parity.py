"""Planner parity: the B200 build's search must select byte-identical plans.

Golden vectors were produced by the REFERENCE planner
(tests/golden/make_planner_golden.py); this file never imports the reference.
"""

import hashlib
import json
from pathlib import Path

import pytest

from paper_2504_21411_b200.planner import cli, pipesim, profiles, search
from paper_2504_21411_b200.planner.errors import NoFeasiblePlan
from paper_2504_21411_b200.planner.serialize import dumps_canonical

GOLDEN = Path(__file__).parent / "golden"
FIX = GOLDEN / "reference_fixtures"
LINES = [json.loads(l) for l in (GOLDEN / "planner_golden.jsonl").read_text().splitlines()]


def test_cli_reproduces_reference_golden_plan(tmp_path, capsys):
    out = tmp_path / "plan.json"
    for jobs in ("1", "4"):
        rc = cli.main(["search", "--cluster", str(FIX / "cluster_2dev.json"),
                       "--model", str(FIX / "model_2layer.json"),
                       "--training", str(FIX / "training_g8.json"), "--jobs", jobs,
                       "-o", str(out)])
        assert rc == 0
        assert out.read_bytes() == (FIX / "golden_plan.json").read_bytes()
    assert capsys.readouterr().out.startswith("time=0.00088518618794666674 pp=1 microbatch=8")


def test_cli_tiny_memory_is_infeasible(tmp_path, capsys):
    rc = cli.main(["search", "--cluster", str(FIX / "cluster_tiny_memory.json"),
                   "--model", str(FIX / "model_2layer.json"),
                   "--training", str(FIX / "training_g8.json"), "-o", str(tmp_path / "p.json")])
    assert rc == 4
    err = capsys.readouterr().err
    assert "stage" in err and "budget" in err


@pytest.mark.parametrize("doc", LINES, ids=[d["tag"] for d in LINES])
def test_search_matches_reference(doc):
    cluster = profiles.cluster_from_dict(doc["cluster"])
    model = profiles.model_from_dict(doc["model"])
    training = profiles.training_from_dict(doc["training"])
    knobs = doc["knobs"]
    cfg = search.SearchConfig(transitions=knobs["transitions"],
                              memory_buckets=knobs["memory_buckets"])
    if "infeasible" in doc:
        with pytest.raises(NoFeasiblePlan) as err:
            search.optimize(model, cluster, training, cfg)
        exp = doc["infeasible"]
        assert str(err.value) == exp["message"]
        assert err.value.stage_index == exp["stage_index"]
        assert err.value.min_achievable_bytes == exp["min_achievable_bytes"]
        assert err.value.budget_bytes == exp["budget_bytes"]
        return
    rep = search.optimize_with_report(model, cluster, training, cfg)
    assert dumps_canonical(rep.plan.to_dict(), sort_keys=False) == doc["plan"]
    assert rep.memory_binding == doc["memory_binding"]
    sim = pipesim.simulate(rep.plan, model, cluster, training, transitions=knobs["transitions"])
    assert sim.makespan == doc["sim"]["makespan"]
    assert list(sim.stage_peak_memory) == doc["sim"]["peaks"]
    assert sim.bubble_fraction == doc["sim"]["bubble"]
    assert len(sim.trace) == doc["sim"]["n_events"]
    assert hashlib.sha256(pipesim.trace_to_jsonl(sim).encode()).hexdigest() == \
        doc["sim"]["trace_sha256"]
    bundle = cli.build_report(rep.plan, model, cluster, training,
                              transitions=knobs["transitions"])
    blob = dumps_canonical(bundle, sort_keys=False) + cli.report_to_csv(bundle)
    assert hashlib.sha256(blob.encode()).hexdigest() == doc["report_sha256"]


B200_LINES = [json.loads(l) for l in
              (GOLDEN / "planner_golden_b200.jsonl").read_text().splitlines()]


@pytest.mark.parametrize("doc", B200_LINES, ids=[d["tag"] for d in B200_LINES])
def test_committed_b200_profiles_pick_the_reference_plan(doc):
    """The exact inputs bench.py searches on (committed profiles/*.json, re-scoped to N):
    byte-identical Plan JSON and identical simulated schedule vs the reference planner
    (tests/golden/make_planner_golden.py --committed)."""
    cluster = profiles.cluster_from_dict(doc["cluster"])
    model = profiles.model_from_dict(doc["model"])
    training = profiles.training_from_dict(doc["training"])
    plan = search.optimize(model, cluster, training)
    assert dumps_canonical(plan.to_dict(), sort_keys=False) == doc["plan"]
    sim = pipesim.simulate(plan, model, cluster, training)
    assert sim.makespan == doc["sim"]["makespan"]
    assert list(sim.stage_peak_memory) == doc["sim"]["peaks"]
    assert hashlib.sha256(pipesim.trace_to_jsonl(sim).encode()).hexdigest() == \
        doc["sim"]["trace_sha256"]


def test_committed_golden_covers_the_committed_profiles():
    """The golden inputs are the files bench.py loads (regenerate on recalibration)."""
    import sys
    sys.path.insert(0, str(GOLDEN))
    from make_planner_golden import COMMITTED
    root = GOLDEN.parents[1] / "profiles"
    by_tag = {d["tag"]: d for d in B200_LINES}
    for name, cl_file, _, ns in COMMITTED:
        want = profiles.load_model_profile(str(root / f"b200_model_{name}.json"))
        for n in ns:
            assert profiles.model_from_dict(by_tag[f"committed-{name}-n{n}"]["model"]) == want
