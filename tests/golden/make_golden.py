"""Generate golden vectors from the REAL reference simulator (dicesim).

Run in the build container only (``/root/reference`` does not exist on the GPU
box): ``python tests/golden/make_golden.py``. The outputs (``*.npz`` + ``*.json``
next to this script) are committed and are what the oracle and the CUDA path
are checked against. The reference is imported read-only from
``/root/reference/pkg/src``; nothing from it is copied into the repo.
"""
from __future__ import annotations

import json
import math
import os
import sys
import time

import numpy as np

REF = os.environ.get("DICE_REFERENCE_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)

import dicesim as ds                      # noqa: E402
from dicesim import model as dm           # noqa: E402
from dicesim import policies as dp        # noqa: E402
from dicesim import cluster as dc         # noqa: E402
from dicesim.oracle import random_grid    # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden_patterns import fresh_pattern  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def cfg_dict(cfg):
    return {k: (float(v) if isinstance(v, float) else v) for k, v in cfg.__dict__.items()}


def pol_dict(p):
    return dict(sync_strategy=p.sync_strategy.value,
                explicit_layers=None if p.explicit_layers is None else sorted(p.explicit_layers),
                cond_strategy=p.cond_strategy.value, refresh_interval=p.refresh_interval,
                cond_seed=p.cond_seed, warmup=p.warmup,
                period=None if math.isinf(p.period) else int(p.period),
                strict_refresh=p.strict_refresh)


def kat():
    out = {}
    out["sm0_first"] = dm.splitmix64(0, 1)
    out["sm123_100"] = dm.splitmix64(123, 100)
    out["sm_big"] = dm.splitmix64(0xDEADBEEFCAFEF00D, 4096)
    keys = np.array([0, 1, 7, 2 ** 63 + 5, 0xD1CE0B5E55ED5EED, 2 ** 64 - 1], dtype=np.uint64)
    out["mix64_keys"] = keys
    out["mix64_vals"] = np.array([dm.mix64(int(k)) for k in keys], dtype=np.uint64)
    out["uniform_025"] = dm.bits_to_uniform(dm.splitmix64(5, 1000), 0.25)
    out["random_keep"] = dp.random_keep_slots(9, 2, 5, 257, 3)
    np.savez_compressed(os.path.join(HERE, "kat.npz"), **out)


def init_and_layers():
    cfg = ds.ModelConfig(num_layers=2, num_experts=4, num_shared=2, top_k=2, hidden_dim=6,
                         expert_dim=5, num_tokens=3, batch=1, num_steps=4)
    model = ds.init_model(cfg, seed=7)
    out = {}
    for l, lw in enumerate(model.layers):
        out[f"l{l}_w_mix"] = lw.w_mix
        out[f"l{l}_w_gate"] = lw.w_gate
        for e, (w1, w2) in enumerate(lw.experts):
            out[f"l{l}_e{e}_w1"] = w1
            out[f"l{l}_e{e}_w2"] = w2
        for s, (w1, w2) in enumerate(lw.shared):
            out[f"l{l}_s{s}_w1"] = w1
            out[f"l{l}_s{s}_w2"] = w2
    out["x0"] = ds.sample_x0(cfg, 7).values
    # layer ops on seeded inputs
    rng = np.random.default_rng(11)
    tokens = rng.normal(size=(9, cfg.hidden_dim))
    blk = ds.ActivationBlock(tokens, 0)
    out["tokens"] = tokens
    for l in range(2):
        route = dm.gate(model, l, blk)
        out[f"l{l}_ids"], out[f"l{l}_gates"], out[f"l{l}_scores"] = (
            route.expert_ids, route.gates, route.scores)
        out[f"l{l}_local"] = dm.local_block(model, l, blk).values
        out[f"l{l}_shared"] = dm.shared_forward(model, l, blk)
        out[f"l{l}_rows"] = dm.routed_rows(model, l, tokens, route)
        act = rng.random((9, 2)) < 0.6
        out[f"l{l}_act"] = act
        out[f"l{l}_rows_act"] = dm.routed_rows(model, l, tokens, route, act)
        out[f"l{l}_combine"] = dm.combine_outputs(route, out[f"l{l}_rows"], out[f"l{l}_shared"], route)
        out[f"l{l}_e2"] = dm.expert_forward(model, l, 2, tokens)
    np.savez_compressed(os.path.join(HERE, "tiny_model.npz"), **out)
    with open(os.path.join(HERE, "tiny_model.json"), "w") as f:
        json.dump(cfg_dict(cfg), f, indent=1, sort_keys=True)


def gate_cases():
    out = {}
    # exact ties: equal logits -> ids [0,1], gates [.5,.5] (test_model.py:123-130)
    cfg = ds.ModelConfig(num_layers=1, num_experts=8, num_shared=0, top_k=2, hidden_dim=16,
                         expert_dim=8, num_tokens=64, batch=1, num_steps=1)
    model = ds.init_model(cfg, seed=3)
    rng = np.random.default_rng(5)
    u = rng.normal(size=(64, 16))
    u[0] = 0.0                               # all logits equal -> all scores tie
    u[1] = u[2]                              # identical rows
    r = dm.gate(model, 0, ds.ActivationBlock(u, 0))
    out.update(u=u, w_gate=model.layers[0].w_gate, ids=r.expert_ids, gates=r.gates,
               scores=r.scores)
    for k in (1, 3, 8):
        cfgk = ds.ModelConfig(**{**cfg.__dict__, "top_k": k})
        mk = ds.init_model(cfgk, seed=3)
        rk = dm.gate(mk, 0, ds.ActivationBlock(u, 0))
        out[f"ids_k{k}"], out[f"gates_k{k}"] = rk.expert_ids, rk.gates
    np.savez_compressed(os.path.join(HERE, "gate.npz"), **out)


def cache_sequences():
    """Decide/assemble over 24 steps for every cond strategy (+ strict)."""
    out, meta = {}, []
    rng = np.random.default_rng(21)
    n, k, h, L = 37, 3, 2, 2
    case = 0
    for strat in (dp.CondStrategy.LOW_SCORE, dp.CondStrategy.HIGH_SCORE, dp.CondStrategy.RANDOM):
        for R in (1, 2, 5):
            for strict in (False, True):
                pol = dp.PolicyConfig(cond_strategy=strat, refresh_interval=R, cond_seed=13,
                                      strict_refresh=strict)
                cache = dp.TokenCache(L, n, k, h)
                ids_seq, gates_seq, act_seq, wr_seq, rows_seq, g_seq, force_seq, fresh_seq = (
                    [], [], [], [], [], [], [], [])
                for step in range(24):
                    for layer in range(L):
                        ids = np.stack([rng.permutation(6)[:k] for _ in range(n)])
                        gates = rng.random((n, k))
                        route = ds.RouteDecision(ids.astype(np.int64), gates, np.zeros((n, 6)))
                        force = bool(rng.random() < 0.15)
                        a, w = cache.decide(layer, step, route, pol, force_refresh=force)
                        fresh = fresh_pattern(step, layer, k, n, h) * a.T[:, :, None]
                        rows, g = cache.assemble(layer, fresh, route, a, w)
                        ids_seq.append(ids); gates_seq.append(gates); act_seq.append(a)
                        wr_seq.append(w); rows_seq.append(rows); g_seq.append(g)
                        force_seq.append(force)
                p = f"c{case}_"
                out[p + "ids"] = np.array(ids_seq).astype(np.int8)
                out[p + "gates"] = np.array(gates_seq)
                out[p + "active"] = np.array(act_seq); out[p + "write"] = np.array(wr_seq)
                out[p + "rows"] = np.array(rows_seq).astype(np.float32)   # exact: dyadic values
                out[p + "outg"] = np.array(g_seq); out[p + "force"] = np.array(force_seq)
                meta.append(dict(case=case, policy=pol_dict(pol), n=n, k=k, h=h, layers=L, steps=24))
                case += 1
    np.savez_compressed(os.path.join(HERE, "cache.npz"), **out)
    with open(os.path.join(HERE, "cache.json"), "w") as f:
        json.dump(meta, f, indent=1)


def small_runs():
    """Full runs: fixed SMALL config x strategies x policies, plus a slice of
    the reference's own random_grid (oracle.py:218-265)."""
    small = ds.ModelConfig(num_layers=3, num_experts=4, num_shared=1, top_k=2, hidden_dim=8,
                           expert_dim=16, num_tokens=4, batch=2, num_steps=8, step_size=1e-3)
    cases = []
    pols = [ds.NEUTRAL, ds.PolicyConfig(warmup=2, period=3), ds.dice_policy(),
            ds.PolicyConfig(sync_strategy=ds.SyncStrategy.STAGGERED,
                            cond_strategy=ds.CondStrategy.RANDOM, refresh_interval=2),
            ds.PolicyConfig(sync_strategy=ds.SyncStrategy.EXPLICIT, explicit_layers=frozenset({1}),
                            cond_strategy=ds.CondStrategy.HIGH_SCORE, refresh_interval=3,
                            strict_refresh=True, warmup=1, period=4)]
    for strategy in ds.Strategy:
        for pol in pols:
            for dev in (1, 2, 4):
                cases.append((small, strategy, pol, 7, dev))
    for item in random_grid(48, seed=0):
        cases.append(item)
    out, meta = {}, []
    for i, (cfg, strategy, pol, seed, dev) in enumerate(cases):
        model = ds.init_model(cfg, seed=seed)
        x0 = ds.sample_x0(cfg, seed=seed)
        cl = ds.ClusterConfig(num_devices=dev)
        res = ds.run_sampling(model, x0, strategy, pol, cl, seed, record_inputs=(i < 8),
                              record_routes=(i < 8))
        out[f"r{i}_final"] = res.final.values
        out[f"r{i}_per_step_active"] = np.array(res.per_step_active_pairs)
        out[f"r{i}_staleness"] = np.array([(r.layer, r.used_step, r.generated_step)
                                           for r in res.staleness_records])
        if i < 8:
            out[f"r{i}_inputs"] = np.array(res.step_inputs)
            out[f"r{i}_ids"] = np.array([[r.expert_ids for r in row] for row in res.step_routes])
        meta.append(dict(idx=i, config=cfg_dict(cfg), strategy=strategy.value,
                         policy=pol_dict(pol), seed=seed, devices=dev,
                         dispatch_bytes=res.dispatch_bytes, combine_bytes=res.combine_bytes,
                         peak_buffer_bytes=res.peak_buffer_bytes, active_pairs=res.active_pairs,
                         total_pairs=res.total_pairs,
                         histogram={str(k): v for k, v in res.staleness_histogram().items()}))
    np.savez_compressed(os.path.join(HERE, "runs.npz"), **out)
    with open(os.path.join(HERE, "runs.json"), "w") as f:
        json.dump(meta, f, indent=1)


def placement_bytes():
    out = {}
    rng = np.random.default_rng(4)
    for i in range(12):
        E, D = 8, int(rng.choice([1, 2, 4, 8]))
        n, k = int(rng.integers(1, 40)), int(rng.integers(1, 4))
        pl = dc.build_placement(E, D, n)
        ids = rng.integers(0, E, size=(n, k))
        act = rng.random((n, k)) < 0.7
        route = ds.RouteDecision(ids.astype(np.int64), np.ones((n, k)) / k, np.zeros((n, E)))
        out[f"p{i}_ids"], out[f"p{i}_act"], out[f"p{i}_D"] = ids, act, np.array(D)
        out[f"p{i}_expert_dev"], out[f"p{i}_home"] = pl.expert_device, pl.token_home
        out[f"p{i}_total"] = np.array(dc.plan_all_to_all(route, pl, act, 16, 2))
        for d in ("dispatch", "combine"):
            out[f"p{i}_{d}"] = dc.per_device_bytes(route, pl, act, 16, 2, d)
    np.savez_compressed(os.path.join(HERE, "placement.npz"), **out)


def config1():
    """BASELINE config 1 restated at the S/2-8E2A preset geometry:
    L=12, E=8, S=2, k=2, h=384, e=1536, 256 tokens x batch 4, 10 steps, D=2.
    Stores float32 finals for sync / interweaved / full DICE and a teacher-forcing
    slice (first 32 rows of every layer's MoE input at steps 0 and 9, fp64, sync run)."""
    cfg = ds.ModelConfig(num_layers=12, num_experts=8, num_shared=2, top_k=2, hidden_dim=384,
                         expert_dim=1536, num_tokens=256, batch=4, num_steps=10, step_size=2e-4)
    model = ds.init_model(cfg, seed=0)
    x0 = ds.sample_x0(cfg, seed=0)
    out, meta = {}, {"config": cfg_dict(cfg), "seed": 0, "devices": 2}
    runs = [("sync", ds.Strategy.SYNCHRONOUS, ds.NEUTRAL),
            ("interweaved", ds.Strategy.INTERWEAVED, ds.NEUTRAL),
            ("dice", ds.Strategy.INTERWEAVED, ds.dice_policy())]
    for name, strategy, pol in runs:
        t0 = time.time()
        res = ds.run_sampling(model, x0, strategy, pol, ds.ClusterConfig(num_devices=2), 0,
                              record_inputs=True, record_routes=True)
        meta[name + "_seconds"] = time.time() - t0
        out[name + "_final"] = res.final.values.astype(np.float32)
        if name == "sync":
            out[name + "_u_slice"] = np.array([[res.step_inputs[s][l][:32] for l in range(12)]
                                               for s in (0, 9)])
        out[name + "_ids"] = np.array([[r.expert_ids for r in res.step_routes[s]] for s in (0, 9)]
                                      ).astype(np.int8)
        meta[name] = dict(histogram={str(k): v for k, v in res.staleness_histogram().items()},
                          dispatch_bytes=res.dispatch_bytes, combine_bytes=res.combine_bytes,
                          active_pairs=res.active_pairs, total_pairs=res.total_pairs,
                          peak_buffer_bytes=res.peak_buffer_bytes)
    sync = out["sync_final"].astype(np.float64)
    for name in ("interweaved", "dice"):
        d = out[name + "_final"].astype(np.float64) - sync
        meta[name]["mse_vs_sync"] = float(np.mean(d * d))
        meta[name]["rel_l2_vs_sync"] = float(np.linalg.norm(d) / np.linalg.norm(sync))
    np.savez_compressed(os.path.join(HERE, "config1.npz"), **out)
    with open(os.path.join(HERE, "config1.json"), "w") as f:
        json.dump(meta, f, indent=1)


def xl_width():
    """The XL/2-8E2A layer widths (h=1152, e=4608, E=8, S=2, k=2) at a size the
    fp64 reference runs in seconds: 3 layers, 64 tokens x batch 2, 4 steps, D=2,
    eta=2e-5; synchronous and full DICE (Deep sync + LowScore R=2, W=1, P=3).
    Stores float32 finals, the routing ids of every (step, layer) and the run
    accounting (histograms, bytes, pairs)."""
    cfg = ds.ModelConfig(num_layers=3, num_experts=8, num_shared=2, top_k=2, hidden_dim=1152,
                         expert_dim=4608, num_tokens=64, batch=2, num_steps=4, step_size=2e-5)
    model = ds.init_model(cfg, seed=7)
    x0 = ds.sample_x0(cfg, seed=7)
    out, meta = {}, {"config": cfg_dict(cfg), "seed": 7, "devices": 2}
    runs = [("sync", ds.Strategy.SYNCHRONOUS, ds.NEUTRAL),
            ("dice", ds.Strategy.INTERWEAVED,
             ds.dice_policy(refresh_interval=2, warmup=1, period=3)),
            ("random_strict", ds.Strategy.INTERWEAVED,
             ds.PolicyConfig(sync_strategy=ds.SyncStrategy.STAGGERED,
                             cond_strategy=ds.CondStrategy.RANDOM, refresh_interval=2,
                             strict_refresh=True)),
            ("displaced_high", ds.Strategy.DISPLACED,
             ds.PolicyConfig(sync_strategy=ds.SyncStrategy.SHALLOW,
                             cond_strategy=ds.CondStrategy.HIGH_SCORE, refresh_interval=3,
                             warmup=1))]
    for name, strategy, pol in runs:
        t0 = time.time()
        res = ds.run_sampling(model, x0, strategy, pol, ds.ClusterConfig(num_devices=2), 7,
                              record_routes=True)
        meta[name + "_strategy"] = strategy.value
        meta[name + "_seconds"] = time.time() - t0
        meta[name + "_policy"] = pol_dict(pol)
        out[name + "_final"] = res.final.values.astype(np.float32)
        out[name + "_ids"] = np.array([[r.expert_ids for r in res.step_routes[s]]
                                       for s in range(cfg.num_steps)]).astype(np.int8)
        meta[name] = dict(histogram={str(k): v for k, v in res.staleness_histogram().items()},
                          dispatch_bytes=res.dispatch_bytes, combine_bytes=res.combine_bytes,
                          active_pairs=res.active_pairs, total_pairs=res.total_pairs,
                          peak_buffer_bytes=res.peak_buffer_bytes)
    np.savez_compressed(os.path.join(HERE, "xl_width.npz"), **out)
    with open(os.path.join(HERE, "xl_width.json"), "w") as f:
        json.dump(meta, f, indent=1)


def g_width():
    """The G-16E2A layer widths (h=1664, e=6656, E=16 experts, S=2, k=2; hidden
    padded to 1792 on the GPU) at a size the fp64 reference runs in about a
    minute: 2 layers, 32 tokens x batch 2, 3 steps, D=4, eta=2e-5, full DICE
    (Deep sync + LowScore R=2, W=1, P=2). Float32 finals, ids and accounting."""
    cfg = ds.ModelConfig(num_layers=2, num_experts=16, num_shared=2, top_k=2, hidden_dim=1664,
                         expert_dim=6656, num_tokens=32, batch=2, num_steps=3, step_size=2e-5)
    model = ds.init_model(cfg, seed=11)
    x0 = ds.sample_x0(cfg, seed=11)
    out, meta = {}, {"config": cfg_dict(cfg), "seed": 11, "devices": 4}
    pol = ds.dice_policy(refresh_interval=2, warmup=1, period=2)
    t0 = time.time()
    res = ds.run_sampling(model, x0, ds.Strategy.INTERWEAVED, pol, ds.ClusterConfig(num_devices=4),
                          11, record_routes=True)
    meta["dice_seconds"] = time.time() - t0
    meta["dice_policy"] = pol_dict(pol)
    out["dice_final"] = res.final.values.astype(np.float32)
    out["dice_ids"] = np.array([[r.expert_ids for r in res.step_routes[s]]
                                for s in range(cfg.num_steps)]).astype(np.int8)
    meta["dice"] = dict(histogram={str(k): v for k, v in res.staleness_histogram().items()},
                        dispatch_bytes=res.dispatch_bytes, combine_bytes=res.combine_bytes,
                        active_pairs=res.active_pairs, total_pairs=res.total_pairs,
                        peak_buffer_bytes=res.peak_buffer_bytes)
    np.savez_compressed(os.path.join(HERE, "g_width.npz"), **out)
    with open(os.path.join(HERE, "g_width.json"), "w") as f:
        json.dump(meta, f, indent=1)


def similarity():
    """step_similarity (model.py:308-346) of the reference's own recorded MoE
    inputs and routes: config 1 (S/2-8E2A widths, D=2; synchronous and full
    DICE) and the reference's xl-toy preset (synchronous, D=4, the acceptance
    criterion 9 trajectory, test_acceptance.py:282-293)."""
    out, meta = {}, {}
    c1 = ds.ModelConfig(num_layers=12, num_experts=8, num_shared=2, top_k=2, hidden_dim=384,
                        expert_dim=1536, num_tokens=256, batch=4, num_steps=10, step_size=2e-4)
    xl = ds.preset("xl-toy")
    cases = [("c1_sync", c1, ds.Strategy.SYNCHRONOUS, ds.NEUTRAL, 2),
             ("c1_dice", c1, ds.Strategy.INTERWEAVED, ds.dice_policy(), 2),
             ("xltoy_sync", xl, ds.Strategy.SYNCHRONOUS, ds.NEUTRAL, 4)]
    for name, cfg, strategy, pol, dev in cases:
        model = ds.init_model(cfg, seed=0)
        res = ds.run_sampling(model, ds.sample_x0(cfg, seed=0), strategy, pol,
                              ds.ClusterConfig(num_devices=dev), 0, record_inputs=True,
                              record_routes=True)
        sim = dm.step_similarity(res.step_inputs, res.step_routes)
        out[name + "_cosine"] = sim.per_layer_cosine
        out[name + "_agreement"] = sim.per_layer_agreement
        meta[name] = dict(config=cfg_dict(cfg), strategy=strategy.value, policy=pol_dict(pol),
                          devices=dev, mean_cosine=sim.mean_cosine,
                          mean_agreement=sim.mean_agreement)
    np.savez_compressed(os.path.join(HERE, "similarity.npz"), **out)
    with open(os.path.join(HERE, "similarity.json"), "w") as f:
        json.dump(meta, f, indent=1)


if __name__ == "__main__":
    which = sys.argv[1:] or ["kat", "init", "gate", "cache", "runs", "placement", "config1",
                             "xl_width", "g_width", "similarity"]
    fns = dict(similarity=similarity, kat=kat, init=init_and_layers, gate=gate_cases, cache=cache_sequences,
               runs=small_runs, placement=placement_bytes, config1=config1, xl_width=xl_width,
               g_width=g_width)
    for w in which:
        t0 = time.time()
        fns[w]()
        print(f"{w}: {time.time() - t0:.1f}s", flush=True)
