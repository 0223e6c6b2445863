"""CPU-only checks: the C-ABI library loads and exports every symbol the
header declares (no compute calls), host-side policy/config/placement logic
against the oracle, and the schedule engine's host control flow (staleness
records, buffer peaks, dispatch/combine logs) against the reference's golden
runs with the device ops stubbed out."""
import json
import math
import os
import re

import numpy as np
import pytest
import torch

import paper_2411_16786_b200 as D
from oracle import dice_oracle as O
from paper_2411_16786_b200 import _lib, cluster, ops, policies

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "tests", "golden")
HEADER = os.path.join(ROOT, "include", "dice_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(?:int|int64_t)\s+(dice_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import ctypes
    if not os.path.exists(_lib.LIB_PATH):
        import build
        build.build()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 18
    for name in syms:
        assert hasattr(lib, name), name
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)
    assert lib.dice_version() == 100


def test_permute_sizing_helpers():
    lib = _lib.load()
    rows = lib.dice_permute_max_rows(8192, 2, 8)
    assert rows % 256 == 0 and rows >= 8192 * 2 + 8 * 255
    # per-block expert counts of the counting pass (blocks of 1024 pairs)
    assert lib.dice_permute_scratch_ints(8192, 2, 8) == 16 * 8
    assert lib.dice_permute_scratch_ints(1 << 20, 2, 8) == 2048 * 8


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "nope.so"))
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(D.NativeLibraryError):
        _lib.load()


def test_error_mapping():
    with pytest.raises(D.ContractError):
        _lib.check(1, "x")
    with pytest.raises(D.ConfigurationError):
        _lib.check(2, "x")
    with pytest.raises(D.NumericsError):
        _lib.check(3, "x")
    with pytest.raises(D.NativeLibraryError):
        _lib.check(4, "x")
    _lib.check(0, "x")


# --------------------------------------------------------------- config / policy
def test_model_config_validation_and_presets():
    with pytest.raises(D.ConfigurationError):
        D.ModelConfig(num_layers=0)
    with pytest.raises(D.ConfigurationError):
        D.ModelConfig(top_k=9, num_experts=8)
    with pytest.raises(D.ConfigurationError):
        D.ModelConfig(step_size=0.0)
    with pytest.raises(D.ConfigurationError):
        D.preset("nope")
    xl = D.preset("xl2-8e2a")
    assert (xl.num_layers, xl.num_experts, xl.hidden_dim, xl.expert_dim) == (28, 8, 1152, 4608)
    assert D.preset("xl-toy").num_layers == 28 and D.preset("g-toy").num_experts == 16


def test_policy_validation_and_sets():
    with pytest.raises(D.ConfigurationError):
        D.PolicyConfig(refresh_interval=0)
    with pytest.raises(D.ConfigurationError):
        D.PolicyConfig(period=2.5)
    with pytest.raises(D.ConfigurationError):
        D.PolicyConfig(sync_strategy=D.SyncStrategy.EXPLICIT)
    p = D.dice_policy()
    assert (p.refresh_interval, p.warmup, p.period) == (5, 6, 10)
    for strat in D.SyncStrategy:
        for L in (1, 4, 7, 28):
            ex = frozenset({0, L - 1}) if strat is D.SyncStrategy.EXPLICIT else None
            assert D.select_sync_layers(strat, L, ex) == O.sync_layer_set(strat.value, L, ex)
    for step in range(40):
        for w, per in ((0, math.inf), (6, 10), (2, 3), (3, 1)):
            assert D.is_sync_step(step, w, per) == O.sync_step(step, w, per)


def test_random_keep_key_matches_oracle():
    for seed, layer, step in ((0, 0, 0), (9, 2, 5), (2 ** 31 - 1, 27, 49)):
        assert policies.random_keep_key(seed, layer, step) == O.random_keep_key(seed, layer, step)
    assert D.model.mix64(123) == O.mix64_int(123)


def test_placement_and_bytes_vs_golden():
    z = np.load(os.path.join(G, "placement.npz"))
    for i in range(12):
        Dn = int(z[f"p{i}_D"])
        ids, act = z[f"p{i}_ids"], z[f"p{i}_act"]
        pl = cluster.build_placement(8, Dn, ids.shape[0])
        assert pl.expert_device.tolist() == z[f"p{i}_expert_dev"].tolist()
        assert pl.token_home.tolist() == z[f"p{i}_home"].tolist()
        route = D.RouteDecision(torch.tensor(ids), torch.ones(ids.shape), torch.zeros(ids.shape[0], 8))
        assert cluster.plan_all_to_all(route, pl, torch.tensor(act), 16, 2) == int(z[f"p{i}_total"])
        for d in ("dispatch", "combine"):
            got = cluster.per_device_bytes(route, pl, torch.tensor(act), 16, 2, d)
            assert got.tolist() == z[f"p{i}_{d}"].tolist()
    with pytest.raises(D.ConfigurationError):
        cluster.build_placement(6, 4, 8)


def test_shard_rows_partition():
    for R in (7, 8, 1024, 8193):
        for Dn in (1, 2, 4, 8):
            homes = (np.arange(R) * Dn) // R
            for d in range(Dn):
                a, b = cluster.shard_rows(R, Dn, d)
                assert np.all(homes[a:b] == d) and (homes == d).sum() == b - a


# ------------------------------------------------- engine host control flow
class _FakeOps:
    """Stand-in for the CUDA ops so the runner's host-side schedule logic runs
    on CPU; values are not computed (test of control flow only)."""

    def __getattr__(self, name):
        return getattr(ops, name)

    @staticmethod
    def permute_max_rows(n, k, E):
        return ((n * k + 255 * E + 255) // 256) * 256

    @staticmethod
    def permute_scratch_ints(n, k, E):
        return max(1, (n * k + 1023) // 1024) * E

    def _noop(self, *a, **k):
        return None

    status_reset = splitmix_fill = gate_topk = cond_decide = route_permute = _noop
    grouped_ffn = cache_assemble = gemm = combine = denoise = pack_rows = _noop
    expert_gemm1_with_shared = expert_gemm2 = expert_gemm2_pairs = _noop
    gemm_consume = consume_rows = gate_route = _noop

    @staticmethod
    def route_state_words(n):
        return 5


def _cpu_model(cfg):
    hp, ep = ops.pad_hidden(cfg.hidden_dim), ops.pad64(cfg.expert_dim)
    E, S = cfg.num_experts, cfg.num_shared
    bf = torch.bfloat16
    layers = [D.model.LayerWeights(torch.zeros(hp, hp, dtype=bf), torch.zeros(E, hp),
                                   torch.zeros(E * ep, hp, dtype=bf), torch.zeros(E * hp, ep, dtype=bf),
                                   torch.zeros(S * ep, hp, dtype=bf) if S else None,
                                   torch.zeros(hp, S * ep, dtype=bf) if S else None)
              for _ in range(cfg.num_layers)]
    return D.ToyModel(config=cfg, seed=0, layers=layers, experts=(0, E), hp=hp, ep=ep, device="cpu")


RUNS = json.load(open(os.path.join(G, "runs.json")))


@pytest.mark.parametrize("idx", range(len(RUNS)))
def test_runner_control_flow_vs_reference(idx, monkeypatch):
    from paper_2411_16786_b200 import schedules
    fake = _FakeOps()
    monkeypatch.setattr(schedules, "ops", fake)
    monkeypatch.setattr(policies, "ops", fake)
    m = RUNS[idx]
    z = np.load(os.path.join(G, "runs.npz"))
    cfg = D.ModelConfig(**m["config"])
    d = m["policy"]
    pol = D.PolicyConfig(sync_strategy=D.SyncStrategy(d["sync_strategy"]),
                         explicit_layers=None if d["explicit_layers"] is None else frozenset(d["explicit_layers"]),
                         cond_strategy=D.CondStrategy(d["cond_strategy"]),
                         refresh_interval=d["refresh_interval"], cond_seed=d["cond_seed"],
                         warmup=d["warmup"], period=math.inf if d["period"] is None else d["period"],
                         strict_refresh=d["strict_refresh"])
    x0 = D.ActivationBlock(torch.zeros(cfg.total_rows, cfg.hidden_dim), 0)
    r = schedules.DeviceRunner(_cpu_model(cfg), x0, D.Strategy(m["strategy"]), pol,
                               D.ClusterConfig(num_devices=m["devices"]), m["seed"])
    r._reset_state()
    for step in range(cfg.num_steps):
        r._run_step(step)
    got = np.array([(s.layer, s.used_step, s.generated_step) for s in r.records])
    assert np.array_equal(got, z[f"r{idx}_staleness"])
    assert r.peak_buffer_bytes == m["peak_buffer_bytes"]
    # every dispatch is processed once, except displaced re-processing / leftovers
    assert len(r.dispatch_log) == cfg.num_steps * cfg.num_layers
    if m["strategy"] != "displaced":
        assert sorted(r.combine_log) == sorted(r.dispatch_log)


def test_runner_rejects_bad_inputs():
    cfg = D.ModelConfig(num_layers=2, num_experts=4, hidden_dim=8, expert_dim=16, num_tokens=4,
                        batch=1, num_steps=2)
    model = _cpu_model(cfg)
    with pytest.raises(D.ContractError):
        D.DeviceRunner(model, D.ActivationBlock(torch.zeros(4, 8), 3), D.Strategy.SYNCHRONOUS,
                       D.NEUTRAL, D.ClusterConfig(num_devices=1), 0)
    with pytest.raises(D.ContractError):
        D.DeviceRunner(model, D.ActivationBlock(torch.zeros(3, 8), 0), D.Strategy.SYNCHRONOUS,
                       D.NEUTRAL, D.ClusterConfig(num_devices=1), 0)
    with pytest.raises(D.ContractError):
        D.DeviceRunner(model, D.ActivationBlock(torch.zeros(4, 8), 0), "displaced",
                       D.NEUTRAL, D.ClusterConfig(num_devices=1), 0)


def test_pad_hidden_rule():
    # multiples of 192 / 256 keep the 64-padding; others go to 256 when <= 10 % more
    assert [ops.pad_hidden(h) for h in (32, 128, 384, 1152, 1664, 2048, 1000, 4096)] == \
        [64, 128, 384, 1152, 1792, 2048, 1024, 4096]
