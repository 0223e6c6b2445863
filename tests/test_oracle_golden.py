"""Pin the CPU oracle (oracle/dice_oracle.py) to golden vectors produced by the
real reference (tests/golden/make_golden.py). CPU only."""
import json
import math
import os

import numpy as np
import pytest

from oracle import dice_oracle as O

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(G, name))


def policy_of(d):
    return O.Policy(sync_strategy=d["sync_strategy"],
                    explicit_layers=None if d["explicit_layers"] is None
                    else frozenset(d["explicit_layers"]),
                    cond_strategy=d["cond_strategy"], refresh_interval=d["refresh_interval"],
                    cond_seed=d["cond_seed"], warmup=d["warmup"],
                    period=math.inf if d["period"] is None else d["period"],
                    strict_refresh=d["strict_refresh"])


def test_splitmix_known_answers():
    k = load("kat.npz")
    assert int(O.stream_bits(0, 0, 1)[0]) == 0xE220A8397B1DCDAF      # test_model.py:36
    assert np.array_equal(O.stream_bits(0, 0, 1), k["sm0_first"])
    assert np.array_equal(O.stream_bits(123, 0, 100), k["sm123_100"])
    big = k["sm_big"]
    seed = 0xDEADBEEFCAFEF00D
    assert np.array_equal(O.stream_bits(seed, 0, 4096), big)
    assert np.array_equal(O.stream_bits(seed, 1000, 77), big[1000:1077])   # counter-based offset
    for key, val in zip(k["mix64_keys"], k["mix64_vals"]):
        assert O.mix64_int(int(key)) == int(val)
    assert np.array_equal(O.to_uniform(O.stream_bits(5, 0, 1000), 0.25), k["uniform_025"])
    assert np.array_equal(O.random_keep(9, 2, 5, 257, 3), k["random_keep"])


def tiny():
    cfg = json.load(open(os.path.join(G, "tiny_model.json")))
    return O.Geometry(**cfg), load("tiny_model.npz")


def test_streamed_init_matches_reference_weights():
    g, z = tiny()
    params = O.init_params(g, 7)
    for l, p in enumerate(params):
        assert np.array_equal(p.w_mix, z[f"l{l}_w_mix"])
        assert np.array_equal(p.w_gate, z[f"l{l}_w_gate"])
        for e, (w1, w2) in enumerate(p.experts):
            assert np.array_equal(w1, z[f"l{l}_e{e}_w1"]) and np.array_equal(w2, z[f"l{l}_e{e}_w2"])
        for s, (w1, w2) in enumerate(p.shared):
            assert np.array_equal(w1, z[f"l{l}_s{s}_w1"]) and np.array_equal(w2, z[f"l{l}_s{s}_w2"])
    assert np.array_equal(O.initial_latent(g, 7), z["x0"])


def test_layer_ops_bit_exact():
    g, z = tiny()
    params = O.init_params(g, 7)
    tok = z["tokens"]
    for l in range(2):
        p = params[l]
        r = O.route_tokens(tok, p.w_gate, g.top_k)
        assert np.array_equal(r.ids, z[f"l{l}_ids"])
        assert np.array_equal(r.gates, z[f"l{l}_gates"])
        assert np.array_equal(r.scores, z[f"l{l}_scores"])
        assert np.array_equal(O.mixing_block(p, tok), z[f"l{l}_local"])
        assert np.array_equal(O.shared_sum(p, tok), z[f"l{l}_shared"])
        assert np.array_equal(O.expert_rows(p, tok, r), z[f"l{l}_rows"])
        assert np.array_equal(O.expert_rows(p, tok, r, z[f"l{l}_act"]), z[f"l{l}_rows_act"])
        assert np.array_equal(O.weighted_combine(z[f"l{l}_rows"], z[f"l{l}_shared"], r.gates),
                              z[f"l{l}_combine"])
        assert np.array_equal(O.mlp(tok, *p.experts[2]), z[f"l{l}_e2"])


def test_gate_ties_and_topk():
    z = load("gate.npz")
    r = O.route_tokens(z["u"], z["w_gate"], 2)
    assert r.ids[0].tolist() == [0, 1]                          # test_model.py:123-130
    assert np.array_equal(r.ids, z["ids"]) and np.array_equal(r.gates, z["gates"])
    assert np.array_equal(r.scores, z["scores"])
    for k in (1, 3, 8):
        rk = O.route_tokens(z["u"], z["w_gate"], k)
        assert np.array_equal(rk.ids, z[f"ids_k{k}"]) and np.array_equal(rk.gates, z[f"gates_k{k}"])


def test_gate_scalar_softmax_known_answer():
    w = np.zeros((4, 4))
    w[0, 0] = 1.0
    r = O.route_tokens(np.eye(4)[:1], w, 2)
    assert round(r.gates[0, 0], 4) == 0.7311 and round(r.gates[0, 1], 4) == 0.2689


def test_cadence_cache_sequences():
    z = load("cache.npz")
    meta = json.load(open(os.path.join(G, "cache.json")))
    from tests.golden.make_golden_patterns import fresh_pattern
    for m in meta:
        p = f"c{m['case']}_"
        pol = policy_of(m["policy"])
        n, k, h, L = m["n"], m["k"], m["h"], m["layers"]
        cache = O.CadenceCache(L, n, k, h)
        i = 0
        for step in range(m["steps"]):
            for layer in range(L):
                ids = z[p + "ids"][i].astype(np.int64)
                gates = z[p + "gates"][i]
                a, w = cache.decide(layer, step, ids, pol, bool(z[p + "force"][i]))
                assert np.array_equal(a, z[p + "active"][i]), (m["case"], step, layer)
                assert np.array_equal(w, z[p + "write"][i])
                fresh = fresh_pattern(step, layer, k, n, h) * a.T[:, :, None]
                rows, g = cache.assemble(layer, fresh, O.Route(ids, gates, None), a, w)
                assert np.array_equal(rows.astype(np.float32), z[p + "rows"][i])
                assert np.array_equal(g, z[p + "outg"][i])
                i += 1


def test_placement_and_bytes():
    z = load("placement.npz")
    for i in range(12):
        D = int(z[f"p{i}_D"])
        ids, act = z[f"p{i}_ids"], z[f"p{i}_act"]
        ed, home = O.placement(8, D, ids.shape[0])
        assert np.array_equal(ed, z[f"p{i}_expert_dev"]) and np.array_equal(home, z[f"p{i}_home"])
        assert O.remote_pair_bytes(ids, act, ed, home, 16) == int(z[f"p{i}_total"])
        for d in ("dispatch", "combine"):
            assert np.array_equal(O.device_pair_bytes(ids, act, ed, home, 16, 2, d, D),
                                  z[f"p{i}_{d}"])


RUNS = json.load(open(os.path.join(G, "runs.json")))


@pytest.mark.parametrize("idx", range(len(RUNS)))
def test_schedule_runs_bit_exact(idx):
    m = RUNS[idx]
    z = load("runs.npz")
    g = O.Geometry(**m["config"])
    params = O.init_params(g, m["seed"])
    x0 = O.initial_latent(g, m["seed"])
    res = O.run_schedule(g, params, x0, m["strategy"], policy_of(m["policy"]), m["devices"],
                         m["seed"], record=idx < 8)
    assert np.array_equal(res.final, z[f"r{idx}_final"])
    assert np.array_equal(np.array(res.staleness), z[f"r{idx}_staleness"])
    assert {str(k): v for k, v in res.histogram().items()} == m["histogram"]
    assert res.dispatch_bytes == m["dispatch_bytes"]
    assert res.combine_bytes == m["combine_bytes"]
    assert res.peak_buffer_bytes == m["peak_buffer_bytes"]
    assert (res.active_pairs, res.total_pairs) == (m["active_pairs"], m["total_pairs"])
    assert np.array_equal(np.array(res.per_step_active), z[f"r{idx}_per_step_active"])
    if idx < 8:
        assert np.array_equal(np.array(res.inputs), z[f"r{idx}_inputs"])
        assert np.array_equal(np.array([[r.ids for r in row] for row in res.routes]),
                              z[f"r{idx}_ids"])


def test_divergence_reports_step():
    g = O.Geometry(num_layers=3, num_experts=4, num_shared=1, top_k=2, hidden_dim=8,
                   expert_dim=16, num_tokens=4, batch=2, num_steps=8, step_size=1e150)
    with np.errstate(all="ignore"), pytest.raises((O.DivergedAt, O.NonFinite)):
        O.run_schedule(g, O.init_params(g, 7), O.initial_latent(g, 7), O.SYNC, O.Policy(), 2, 7)


def test_gate_weight_matches_full_init():
    g, z = tiny()
    for l in range(2):
        assert np.array_equal(O.gate_weight(g, 7, l), z[f"l{l}_w_gate"])


XL_POLICIES = {"sync": (O.SYNC, O.Policy()),
               "dice": (O.INTERWEAVED, O.dice_defaults(refresh_interval=2, warmup=1, period=3)),
               "random_strict": (O.INTERWEAVED, O.Policy(sync_strategy=O.SYNC_STAGGERED,
                                                         cond_strategy=O.COND_RANDOM,
                                                         refresh_interval=2, strict_refresh=True)),
               "displaced_high": (O.DISPLACED, O.Policy(sync_strategy=O.SYNC_SHALLOW,
                                                        cond_strategy=O.COND_HIGH,
                                                        refresh_interval=3, warmup=1))}


def test_xl_width_runs_match_reference():
    """The oracle at the XL/2-8E2A layer widths (h=1152, e=4608; 3 layers, 128
    rows, 4 steps) against the real reference's runs: finals to the fp32 storage
    rounding of the fixture, identical staleness histograms, pairs and bytes."""
    meta = json.load(open(os.path.join(G, "xl_width.json")))
    z = np.load(os.path.join(G, "xl_width.npz"))
    g = O.Geometry(**meta["config"])
    params = O.init_params(g, meta["seed"])
    x0 = O.initial_latent(g, meta["seed"])
    for name, (strategy, pol) in XL_POLICIES.items():
        r = O.run_schedule(g, params, x0, strategy, pol, meta["devices"], meta["seed"])
        ref = z[name + "_final"].astype(np.float64)
        assert np.abs(r.final - ref).max() <= 1e-6 * max(1.0, np.abs(ref).max())
        m = meta[name]
        assert {str(k): v for k, v in r.histogram().items()} == m["histogram"]
        assert (r.active_pairs, r.total_pairs) == (m["active_pairs"], m["total_pairs"])
        assert (r.dispatch_bytes, r.combine_bytes) == (m["dispatch_bytes"], m["combine_bytes"])
        assert r.peak_buffer_bytes == m["peak_buffer_bytes"]


def test_step_similarity_matches_reference():
    """f3: the oracle's step_similarity (model.py:316-346) on its own recorded
    xl-toy synchronous trajectory reproduces the reference's per-layer cosines
    and top-1 agreements (tests/golden/similarity.*, make_golden.similarity)."""
    meta = json.load(open(os.path.join(G, "similarity.json")))["xltoy_sync"]
    gold = load("similarity.npz")
    c = meta["config"]
    g = O.Geometry(**{k: c[k] for k in ("num_layers", "num_experts", "num_shared", "top_k",
                                        "hidden_dim", "expert_dim", "num_tokens", "batch",
                                        "num_steps", "step_size")})
    res = O.run_schedule(g, O.init_params(g, 0), O.initial_latent(g, 0), O.SYNC, O.Policy(),
                         meta["devices"], 0, record=True)
    cos, agree = O.step_similarity(res.inputs, res.routes)
    assert np.allclose(cos, gold["xltoy_sync_cosine"], rtol=0, atol=1e-13)
    assert np.array_equal(agree, gold["xltoy_sync_agreement"])
    assert abs(float(np.mean(cos)) - meta["mean_cosine"]) < 1e-13
