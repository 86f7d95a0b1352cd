"""CPU tests of the runtime's host-side logic: C-ABI exports, rank topology, reshard
plans (pure and executed over a gloo world of 2/4 processes), the 1F1B op order."""

import itertools
import os
import re
import socket
from pathlib import Path

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_21411_b200.planner.pipesim import one_f_one_b_order
from paper_2504_21411_b200.runtime.reshard import Layout, index_tensors, plan_transition
from paper_2504_21411_b200.runtime.topology import dp_members, tp_members

ROOT = Path(__file__).resolve().parents[1]


def test_library_exports_every_header_symbol():
    import ctypes
    from paper_2504_21411_b200 import kernels
    lib_path = kernels.LIB_PATH
    if not lib_path.exists():
        from paper_2504_21411_b200.build import build
        build()
    header = (ROOT / "include" / "galv.h").read_text()
    declared = sorted(set(re.findall(r"\b(galv_[a-z0-9_]+)\s*\(", header)))
    assert len(declared) >= 25
    lib = ctypes.CDLL(str(lib_path))
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert set(declared) <= set(kernels.EXPORTED), set(declared) - set(kernels.EXPORTED)
    lib.galv_abi_version.restype = ctypes.c_int32
    assert lib.galv_abi_version() == 1


def test_kernels_refuse_cpu_tensors():
    from paper_2504_21411_b200 import kernels as K
    with pytest.raises(RuntimeError):
        K.gemm(torch.zeros(8, 8), torch.zeros(8, 8))


def test_topology_members_contiguous():
    # stage 1 of a 2-stage, 8-device-per-stage layout, tp=2
    assert tp_members(1, 8, 2, 3) == [14, 15]
    assert dp_members(1, 8, 2, 1) == [9, 11, 13, 15]
    assert dp_members(0, 4, 4, 2) == [2]


LAYOUTS = {n: [Layout(tp, n // tp, sp) for tp in (1, 2, 4, 8) if tp <= n
               for sp in (False, True) if not (sp and tp == 1)] for n in (1, 2, 4, 8)}


@pytest.mark.parametrize("n", [2, 4, 8])
def test_reshard_plans_cover_every_row_exactly(n):
    T = 64
    data = torch.arange(T)
    for src, dst in itertools.product(LAYOUTS[n], LAYOUTS[n]):
        plan = plan_transition(src, dst, T)
        held = [data[slice(*src.token_range(i, T))] for i in range(n)]
        for j in range(n):
            lo, hi = dst.token_range(j, T)
            out = torch.full((hi - lo,), -1)
            for i in range(n):
                s, r = plan.send_rows[i][j], plan.recv_rows[j][i]
                assert s[1] - s[0] == r[1] - r[0]
                out[r[0]:r[1]] = held[i][s[0]:s[1]]
            assert torch.equal(out, data[lo:hi]), (src, dst, j)
        # replicas -> their own slices never need the network
        if src.tp == dst.tp * dst.dp and not src.sp and src.dp == 1:
            assert not plan.moves_data


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _reshard_worker(rank, world, port, pairs, T, h):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    full = torch.arange(T * h, dtype=torch.float32).view(T, h)
    for src, dst in pairs:
        plan = plan_transition(src, dst, T)
        sidx, ss, ridx, rs = index_tensors(plan, rank, "cpu")
        x = full[slice(*src.token_range(rank, T))]
        send = x.index_select(0, sidx)                    # pack (galv_gather_rows on GPU)
        recv = torch.empty(sum(rs), h)
        dist.all_to_all_single(recv, send, rs, ss)        # the single collective
        lo, hi = dst.token_range(rank, T)
        out = torch.empty(hi - lo, h)
        out.index_copy_(0, ridx, recv)                    # unpack (galv_scatter_rows on GPU)
        assert torch.equal(out, full[lo:hi]), (rank, src, dst)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_reshard_over_gloo(world):
    pairs = list(itertools.product(LAYOUTS[world], LAYOUTS[world]))
    mp.spawn(_reshard_worker, args=(world, _free_port(), pairs, 32, 8), nprocs=world, join=True)


def _topology_worker(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2504_21411_b200.planner.strategy import ParallelStrategy as PS
    from paper_2504_21411_b200.runtime.config import HybridConfig
    from paper_2504_21411_b200.runtime.topology import Topology
    hc = HybridConfig(pp=1, microbatch=2, n_microbatches=1, stage_ranges=((0, 2),),
                      layer_strategies=(PS(2, 1, 0, False, False), PS(1, 2, 1, False, False)))
    topo = Topology(hc)
    t = torch.tensor([float(rank + 1)])
    from paper_2504_21411_b200.runtime import comm
    comm.all_reduce(t, topo.tp(2))
    assert t.item() == 3.0
    u = torch.tensor([float(rank + 1)])
    comm.all_reduce(u, topo.dp(1))
    assert u.item() == 3.0
    assert topo.tp(1).size == 1 and topo.dp(2).size == 1
    dist.destroy_process_group()


def test_topology_groups_over_gloo():
    mp.spawn(_topology_worker, args=(2, _free_port()), nprocs=2, join=True)


@pytest.mark.parametrize("pp,m", [(1, 4), (2, 4), (4, 8), (4, 2)])
def test_1f1b_order_is_complete_and_causal(pp, m):
    for stage in range(pp):
        ops = one_f_one_b_order(pp, stage, m)
        assert sorted(k for kind, k in ops if kind == "fwd") == list(range(1, m + 1))
        assert sorted(k for kind, k in ops if kind == "bwd") == list(range(1, m + 1))
        seen_f = set()
        live = 0
        for kind, k in ops:
            if kind == "fwd":
                seen_f.add(k)
                live += 1
            else:
                assert k in seen_f
                live -= 1
            assert live <= min(m, pp - stage)


@pytest.mark.parametrize("name", ["tiny-gpt", "gpt2-medium", "gpt-1.3b", "llama2-7b", "llama2-13b"])
def test_embedding_head_fold_accounts_for_the_whole_model(name):
    """profiler.fold_embedding_head: the planned layers' parameters sum to the model's,
    and the cost model's training FLOPs per token (3x fwd, costmodel.py:104-106) equal
    the model's 6*L*P + 12*L*h*s + 6*h*V."""
    from paper_2504_21411_b200.profiler import planned_profile
    from paper_2504_21411_b200.runtime.config import MODEL_PRESETS, profile_for
    cfg = MODEL_PRESETS[name]
    prof = planned_profile(cfg)
    assert sum(lp.param_count for lp in prof.layers) == cfg.total_params()
    fwd = sum(lp.flops_per_token + lp.flops_per_token_sq * cfg.seq_len for lp in prof.layers)
    assert 3.0 * fwd == pytest.approx(cfg.train_flops_per_token(), rel=1e-12)
    base = profile_for(cfg)
    assert prof.layers[1:-1] == base.layers[1:-1]


@pytest.mark.parametrize("name", ["gpt2-medium", "llama2-7b", "llama2-13b"])
def test_committed_model_profiles_carry_the_fold(name):
    import json
    from paper_2504_21411_b200.planner.profiles import load_model_profile
    from paper_2504_21411_b200.profiler import calibrated_model_profile
    from paper_2504_21411_b200.runtime.config import MODEL_PRESETS
    meta = json.loads((ROOT / "profiles" / f"b200_model_{name}.meta.json").read_text())
    prof = load_model_profile(str(ROOT / "profiles" / f"b200_model_{name}.json"))
    assert prof == calibrated_model_profile(MODEL_PRESETS[name], meta["activation"])
    assert sum(lp.param_count for lp in prof.layers) == MODEL_PRESETS[name].total_params()


def _plan_inputs(n=4, mem=180_000_000_000):
    from paper_2504_21411_b200.planner import profiles as P
    from paper_2504_21411_b200.runtime.config import MODEL_PRESETS, profile_for
    cfg = MODEL_PRESETS["gpt2-medium"]
    table = tuple(P.BandwidthEntry("intra_node", g, 7e11, 5e-6) for g in (2, 4) if g <= n)
    cluster = P.ClusterProfile(n, n, 1.2e15, mem, 0.0, table)
    return cfg, profile_for(cfg), cluster, P.TrainingConfig(global_batch=16 * n)


def test_runtime_accepts_a_fresh_searched_plan():
    from paper_2504_21411_b200.planner.search import optimize
    from paper_2504_21411_b200.runtime.config import get_hybrid_parallel_configs
    cfg, mp, cluster, training = _plan_inputs()
    plan = optimize(mp, cluster, training)
    hc = get_hybrid_parallel_configs(plan.to_dict(), cfg, model_profile=mp, cluster=cluster,
                                     training=training)
    assert hc.layer_strategies == tuple(plan.layer_strategies)


def test_runtime_refuses_stale_and_over_budget_plans():
    """ref search.py:823-913 (validate_plan) -- the runtime raises InvalidPlan instead of
    running a plan searched under other profiles (CLI exit 5, cli.py:21-25)."""
    import dataclasses
    from paper_2504_21411_b200.planner.errors import InvalidPlan, ValidationError
    from paper_2504_21411_b200.planner.search import optimize
    from paper_2504_21411_b200.runtime.config import get_hybrid_parallel_configs
    cfg, mp, cluster, training = _plan_inputs()
    plan = optimize(mp, cluster, training)
    # stale: costed under a 2x faster device
    fast = dataclasses.replace(cluster, device_flops=cluster.device_flops * 2)
    with pytest.raises(InvalidPlan) as ei:
        get_hybrid_parallel_configs(plan, cfg, model_profile=mp, cluster=fast,
                                    training=training)
    assert any("predicted" in p or "stale" in p for p in ei.value.problems), ei.value.problems
    # over budget: the same plan on a device with 1 GB
    small = dataclasses.replace(cluster, device_memory_bytes=1_000_000_000)
    with pytest.raises(InvalidPlan) as ei:
        get_hybrid_parallel_configs(plan, cfg, model_profile=mp, cluster=small,
                                    training=training)
    assert any("budget" in p or "memory" in p for p in ei.value.problems), ei.value.problems
    assert isinstance(ei.value, ValidationError)
    # partial profile sets are a usage error
    with pytest.raises(ValidationError):
        get_hybrid_parallel_configs(plan, cfg, cluster=cluster)


def test_measured_report_bundle_and_csv():
    """report.measured_report: the reference build_report bundle (cli.py:213-292) with the
    measured per-layer / per-stage / total columns from layer events."""
    from paper_2504_21411_b200.planner.search import optimize
    from paper_2504_21411_b200.report import COLUMNS, measured_report, report_to_csv
    cfg, mp, cluster, training = _plan_inputs(n=1)
    plan = optimize(mp, cluster, training)
    L = mp.n_layers
    times = []
    for mb in range(plan.n_microbatches):
        for li in range(L):
            times += [("fwd", li, mb, 0.001), ("bwd", li, mb, 0.002)]
        times += [("head", L - 1, mb, 0.0005), ("embed_fwd", 0, mb, 0.0001),
                  ("embed_bwd", 0, mb, 0.0001)]
    b = measured_report(plan, mp, cluster, training, stage=0, layer_times=times,
                        iteration_s=0.5, dp_sync_exposed_s=0.0, peak_memory_bytes=10)
    mid = b["layers"][1]
    assert mid["measured_time_total"] == pytest.approx(0.003)
    assert mid["relative_error"] == pytest.approx((0.003 - mid["time_total"]) / mid["time_total"])
    assert b["layers"][-1]["measured_time_total"] == pytest.approx(0.0035)
    assert b["layers"][0]["measured_time_total"] == pytest.approx(0.0032)
    st = b["stages"][0]
    assert st["measured_per_microbatch_time"] == pytest.approx(0.003 * L + 0.0007)
    assert st["peak_within_prediction"] is True
    assert b["total"]["measured_iteration_time"] == 0.5
    csv = report_to_csv(b).splitlines()
    assert csv[0].split(",") == COLUMNS
    assert len(csv) == 1 + L + plan.pp + 1
    assert all(len(r.split(",")) == len(COLUMNS) for r in csv)


def test_reshard_traffic_within_the_cost_model_bound():
    """a11 (costmodel.py:179-196): the reshard of every layout change of BASELINE config 4's
    alternating TP4 / SDP4 / DP2xTP2 plan sends no more bytes from its busiest rank than the
    all-gather volume the cost model charges for the transition; tp -> dp moves nothing."""
    from paper_2504_21411_b200.planner import profiles as P
    from paper_2504_21411_b200.planner.search import make_plan
    from paper_2504_21411_b200.planner.strategy import ParallelStrategy as PS
    from paper_2504_21411_b200.profiler import planned_profile
    from paper_2504_21411_b200.report import transition_traffic
    from paper_2504_21411_b200.runtime.config import MODEL_PRESETS
    cfg = MODEL_PRESETS["gpt-1.3b"]
    mp = planned_profile(cfg)
    table = tuple(P.BandwidthEntry("intra_node", g, 4e11, 5e-6) for g in (2, 4))
    cluster = P.ClusterProfile(4, 4, 1.2e15, 191_000_000_000, 0.1, table)
    strs = [PS(4, 1, 0, False, False), PS(1, 4, 3, False, False), PS(2, 2, 0, False, False)]
    plan = make_plan(mp, cluster, P.TrainingConfig(global_batch=64), 1, 8,
                     [strs[i % 3] for i in range(cfg.n_layers)])
    tt = transition_traffic(plan, mp, hidden=cfg.hidden)
    assert len(tt) == cfg.n_layers - 1
    for li, t in tt.items():
        assert t["reshard_bytes_max_rank"] <= t["model_allgather_bytes_per_rank"], (li, t)
    assert tt[1]["reshard_bytes_max_rank"] == 0  # TP4 -> DP4: every rank already holds it
