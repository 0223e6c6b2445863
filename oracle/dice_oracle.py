"""CPU oracle for the DICE expert-parallel MoE sampling path — TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product. Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` leg may import it. The shipped path (``paper_2411_16786_b200``)
never calls into it and fails loudly when its CUDA library is missing.

It restates, in float64 numpy, the algorithm of the reference simulator
``dicesim`` (``/root/reference/pkg/src/dicesim``). Each function cites the
reference ``file:line`` it follows. Parity of this restatement is pinned
against golden vectors produced by the real reference
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``,
checked by ``tests/test_oracle_golden.py``).

Differences from the reference that do not change any value:
* weights are generated per layer from the counter-based stream (the
  reference materialises one ``splitmix64(seed, total)`` array, model.py:140);
  position ``p`` of the stream is the same value either way, so XL/G
  geometries fit in memory;
* the schedule engine keeps only the state the three schedules need; the
  alpha-beta timeline (cluster.py:112-216) is out of scope.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
from scipy.special import erf

U64 = 0xFFFFFFFFFFFFFFFF
GAMMA = 0x9E3779B97F4A7C15          # model.py:17
MUL1 = 0xBF58476D1CE4E5B9           # model.py:18
MUL2 = 0x94D049BB133111EB           # model.py:19
X0_TAG = 0xD1CE0B5E55ED5EED         # model.py:23
RANDOM_SLOT_TAG = 0x7C0DD17105A17BAD  # policies.py:18

SYNC, DISPLACED, INTERWEAVED = "synchronous", "displaced", "interweaved"   # schedules.py:42-45
SYNC_NONE, SYNC_DEEP, SYNC_SHALLOW, SYNC_STAGGERED, SYNC_EXPLICIT = (
    "none", "deep", "shallow", "staggered", "explicit")                     # policies.py:21-26
COND_OFF, COND_LOW, COND_HIGH, COND_RANDOM = (
    "off", "low_score", "high_score", "random")                             # policies.py:29-33


# --------------------------------------------------------------------------- PRF
def mix_u64(z: np.ndarray) -> np.ndarray:
    """The two xor-shift-multiply rounds + final xor of splitmix64 (model.py:34-36)."""
    z = (z ^ (z >> np.uint64(30))) * np.uint64(MUL1)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(MUL2)
    return z ^ (z >> np.uint64(31))


def stream_bits(seed: int, start: int, count: int) -> np.ndarray:
    """Outputs ``start .. start+count-1`` (0-based) of splitmix64(seed) (model.py:28-36).

    Output ``p`` uses counter ``p + 1``: z = seed + (p+1)*gamma mod 2^64.
    """
    with np.errstate(over="ignore"):
        ctr = np.arange(start + 1, start + count + 1, dtype=np.uint64)
        z = np.uint64(seed & U64) + ctr * np.uint64(GAMMA)
        return mix_u64(z)


def mix64_int(value: int) -> int:
    """Scalar splitmix64 of one key (model.py:39-44), Python ints mod 2^64."""
    z = (value + GAMMA) & U64
    z = ((z ^ (z >> 30)) * MUL1) & U64
    z = ((z ^ (z >> 27)) * MUL2) & U64
    return z ^ (z >> 31)


def to_uniform(bits: np.ndarray, halfwidth: float) -> np.ndarray:
    """[-a, a) from the top 53 bits (model.py:47-50)."""
    unit = (bits >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return halfwidth * (2.0 * unit - 1.0)


def gelu(x: np.ndarray) -> np.ndarray:
    """Exact erf GELU (model.py:53-55)."""
    return 0.5 * x * (1.0 + erf(x / math.sqrt(2.0)))


# ------------------------------------------------------------------- geometry
@dataclass(frozen=True)
class Geometry:
    """Mirror of ModelConfig's fields (model.py:58-90)."""
    num_layers: int = 28
    num_experts: int = 8
    num_shared: int = 2
    top_k: int = 2
    hidden_dim: int = 32
    expert_dim: int = 64
    num_tokens: int = 16
    batch: int = 4
    num_steps: int = 50
    step_size: float = 2e-4

    @property
    def total_rows(self) -> int:
        return self.num_tokens * self.batch


def layer_value_count(g: Geometry) -> int:
    """Stream values consumed per layer (model.py:126-130)."""
    h, e = g.hidden_dim, g.expert_dim
    return h * h + h * g.num_experts + 2 * h * e * (g.num_experts + g.num_shared)


@dataclass
class LayerParams:
    w_mix: np.ndarray
    w_gate: np.ndarray
    experts: list
    shared: list


def init_layer(g: Geometry, seed: int, layer: int) -> LayerParams:
    """One layer's weights at its stream offset (model.py:133-162 order:
    W_mix, W_gate, routed experts (W1, W2) 0..E-1, shared experts (W1, W2))."""
    h, e = g.hidden_dim, g.expert_dim
    a_h, a_e = float(np.sqrt(1.0 / h)), float(np.sqrt(1.0 / e))
    pos = layer * layer_value_count(g)
    bits = stream_bits(seed, pos, layer_value_count(g))
    cur = 0

    def take(rows, cols, a):
        nonlocal cur
        block = to_uniform(bits[cur:cur + rows * cols], a).reshape(rows, cols)
        cur += rows * cols
        return block

    w_mix = take(h, h, a_h)
    w_gate = take(h, g.num_experts, a_h)
    experts = [(take(h, e, a_h), take(e, h, a_e)) for _ in range(g.num_experts)]
    shared = [(take(h, e, a_h), take(e, h, a_e)) for _ in range(g.num_shared)]
    return LayerParams(w_mix, w_gate, experts, shared)


def gate_weight(g: Geometry, seed: int, layer: int) -> np.ndarray:
    """Only W_gate of one layer, from its stream offset (model.py:157)."""
    h = g.hidden_dim
    start = layer * layer_value_count(g) + h * h
    bits = stream_bits(seed, start, h * g.num_experts)
    return to_uniform(bits, float(np.sqrt(1.0 / h))).reshape(h, g.num_experts)


def init_params(g: Geometry, seed: int) -> list:
    return [init_layer(g, seed, l) for l in range(g.num_layers)]


def initial_latent(g: Geometry, seed: int) -> np.ndarray:
    """x0 uniform in [-1, 1) from the tagged stream (model.py:181-186)."""
    n = g.total_rows * g.hidden_dim
    return to_uniform(stream_bits(mix64_int(seed ^ X0_TAG), 0, n), 1.0).reshape(
        g.total_rows, g.hidden_dim)


# ----------------------------------------------------------------- layer math
@dataclass
class Route:
    ids: np.ndarray      # [n, k] int64
    gates: np.ndarray    # [n, k] f64
    scores: np.ndarray   # [n, E] f64


class NonFinite(Exception):
    pass


def route_tokens(u: np.ndarray, w_gate: np.ndarray, k: int) -> Route:
    """Softmax gate, stable top-k on scores (ties -> lower id), renormalised
    over the k picks (model.py:209-223)."""
    if not np.all(np.isfinite(u)):
        raise NonFinite("non-finite activations entering gate")
    logits = u @ w_gate
    ex = np.exp(logits - logits.max(axis=1, keepdims=True))
    scores = ex / ex.sum(axis=1, keepdims=True)
    ids = np.argsort(-scores, axis=1, kind="stable")[:, :k]
    picked = np.take_along_axis(scores, ids, axis=1)
    return Route(ids.astype(np.int64), picked / picked.sum(axis=1, keepdims=True), scores)


def forced_route(u: np.ndarray, w_gate: np.ndarray, ids: np.ndarray) -> Route:
    """Teacher-forced routing: the given expert ids with gates renormalised
    from this oracle's own softmax scores (model.py:216-222)."""
    logits = u @ w_gate
    ex = np.exp(logits - logits.max(axis=1, keepdims=True))
    scores = ex / ex.sum(axis=1, keepdims=True)
    ids = np.asarray(ids, dtype=np.int64)
    picked = np.take_along_axis(scores, ids, axis=1)
    return Route(ids, picked / picked.sum(axis=1, keepdims=True), scores)


def mlp(x: np.ndarray, w1: np.ndarray, w2: np.ndarray) -> np.ndarray:
    """gelu(x W1) W2 (model.py:226-232)."""
    return gelu(x @ w1) @ w2


def shared_sum(p: LayerParams, u: np.ndarray) -> np.ndarray:
    """Sum of shared MLPs on fresh u, accumulated left to right (model.py:235-241)."""
    out = np.zeros_like(u)
    for w1, w2 in p.shared:
        out += mlp(u, w1, w2)
    return out


def mixing_block(p: LayerParams, h: np.ndarray) -> np.ndarray:
    """gelu(h W_mix) + h (model.py:244-252)."""
    return gelu(h @ p.w_mix) + h


def expert_rows(p: LayerParams, u: np.ndarray, route: Route, active=None) -> np.ndarray:
    """[k, n, h] per-slot expert outputs; groups (slot, expert) in ascending
    token order, inactive pairs stay zero (model.py:255-276)."""
    n, k = route.ids.shape
    rows = np.zeros((k, n, u.shape[1]))
    for s in range(k):
        for ex in range(len(p.experts)):
            sel = route.ids[:, s] == ex
            if active is not None:
                sel &= active[:, s]
            idx = np.flatnonzero(sel)
            if idx.size:
                rows[s, idx] = mlp(u[idx], *p.experts[ex])
    return rows


def weighted_combine(rows: np.ndarray, shared: np.ndarray, gates: np.ndarray) -> np.ndarray:
    """shared + sum_s gates[:, s] * rows[s], slots left to right (model.py:279-298)."""
    out = shared.copy()
    for s in range(rows.shape[0]):
        out += gates[:, s:s + 1] * rows[s]
    return out


# ------------------------------------------------------------------- policies
@dataclass(frozen=True)
class Policy:
    """Mirror of PolicyConfig (policies.py:36-59)."""
    sync_strategy: str = SYNC_NONE
    explicit_layers: frozenset | None = None
    cond_strategy: str = COND_OFF
    refresh_interval: int = 1
    cond_seed: int | None = None
    warmup: int = 0
    period: float = math.inf
    strict_refresh: bool = False


def dice_defaults(refresh_interval=5, warmup=6, period=10) -> Policy:
    """Deep selective sync + LowScore conditional comm (policies.py:65-70)."""
    return Policy(sync_strategy=SYNC_DEEP, cond_strategy=COND_LOW,
                  refresh_interval=refresh_interval, warmup=warmup, period=period)


def sync_layer_set(strategy: str, num_layers: int, explicit=None) -> frozenset:
    """policies.py:73-93."""
    half = -(-num_layers // 2)
    return {
        SYNC_NONE: frozenset(),
        SYNC_DEEP: frozenset(range(half, num_layers)),
        SYNC_SHALLOW: frozenset(range(half)),
        SYNC_STAGGERED: frozenset(range(1, num_layers, 2)),
        SYNC_EXPLICIT: frozenset(int(v) for v in (explicit or ())),
    }[strategy]


def sync_step(step: int, warmup: int, period: float) -> bool:
    """policies.py:96-104."""
    if step < warmup:
        return True
    return period != math.inf and (step - warmup) % int(period) == 0


def random_keep_key(seed: int, layer: int, step: int) -> int:
    """PRF key for the Random strategy's kept slot (policies.py:113-114)."""
    key = mix64_int((mix64_int((seed ^ RANDOM_SLOT_TAG) & U64) + layer) & U64)
    return mix64_int((key + step) & U64)


def random_keep(seed: int, layer: int, step: int, n: int, k: int) -> np.ndarray:
    """policies.py:107-115."""
    return (stream_bits(random_keep_key(seed, layer, step), 0, n) % np.uint64(k)).astype(np.int64)


def reduced_mask(n: int, k: int, strategy: str, seed=0, layer=0, step=0) -> np.ndarray:
    """[n, k] cacheable slots (policies.py:118-139)."""
    m = np.zeros((n, k), dtype=bool)
    if strategy == COND_LOW:
        m[:, 1:] = True
    elif strategy == COND_HIGH:
        m[:, 0] = True
    elif strategy == COND_RANDOM:
        m[:] = True
        m[np.arange(n), random_keep(seed, layer, step, n, k)] = False
    return m


class CadenceCache:
    """Per (layer, token, slot) cached rows/gates/ids + per-token refresh cadence
    (policies.py:142-208)."""

    def __init__(self, layers: int, n: int, k: int, h: int):
        self.rows = np.zeros((layers, k, n, h))
        self.gates = np.zeros((layers, n, k))
        self.ids = np.full((layers, n, k), -1, dtype=np.int64)
        self.last = np.full((layers, n), -(10 ** 9), dtype=np.int64)
        self.mask = np.zeros((layers, n, k), dtype=bool)
        self.primed = np.zeros((layers, n), dtype=bool)

    def decide(self, layer, step, ids, policy: Policy, force=False):
        """Active / cache-write masks; cadence bookkeeping (policies.py:159-186)."""
        n, k = ids.shape
        if policy.cond_strategy == COND_OFF:
            return np.ones((n, k), bool), np.zeros((n, k), bool)
        due = ((step - self.last[layer]) >= policy.refresh_interval) | ~self.primed[layer]
        if force:
            due = np.ones(n, dtype=bool)
        if due.any():
            seed = policy.cond_seed if policy.cond_seed is not None else 0
            fresh = reduced_mask(n, k, policy.cond_strategy, seed, layer, step)
            self.mask[layer][due] = fresh[due]
            self.last[layer][due] = step
            self.primed[layer][due] = True
        red = self.mask[layer]
        active = ~red | due[:, None]
        write = red & due[:, None]
        if policy.strict_refresh:
            moved = red & ~due[:, None] & (ids != self.ids[layer])
            active |= moved
            write |= moved
        return active, write

    def assemble(self, layer, fresh, route: Route, active, write):
        """Merge fresh with cached rows, persist refreshed pairs (policies.py:188-208)."""
        rows = fresh.copy()
        gates = np.where(active, route.gates, self.gates[layer])
        for s in range(fresh.shape[0]):
            stale = ~active[:, s]
            rows[s][stale] = self.rows[layer, s][stale]
            w = write[:, s]
            self.rows[layer, s][w] = fresh[s][w]
        self.gates[layer] = np.where(write, route.gates, self.gates[layer])
        self.ids[layer] = np.where(write, route.ids, self.ids[layer])
        return rows, gates


# ------------------------------------------------------------------- placement
def placement(num_experts: int, devices: int, rows: int):
    """Contiguous expert blocks, near-even contiguous token shards (cluster.py:61-72)."""
    if num_experts % devices:
        raise ValueError("num_experts not divisible by devices")
    expert_dev = np.arange(num_experts) // (num_experts // devices)
    home = (np.arange(rows) * devices) // rows
    return expert_dev, home


def remote_pair_bytes(ids, active, expert_dev, home, h, bpe=2) -> int:
    """Bytes of active pairs whose expert lives off the token's home (cluster.py:82-90)."""
    remote = expert_dev[ids] != home[:, None]
    if active is not None:
        remote &= active
    return int(np.count_nonzero(remote)) * h * bpe


def device_pair_bytes(ids, active, expert_dev, home, h, bpe, direction, devices):
    """Per-device bytes: dispatch at token home, combine at expert device (cluster.py:93-109)."""
    src = np.broadcast_to(home[:, None], ids.shape)
    dst = expert_dev[ids]
    remote = src != dst
    if active is not None:
        remote = remote & active
    origin = src if direction == "dispatch" else dst
    return np.bincount(origin[remote].ravel(), minlength=devices) * h * bpe


# -------------------------------------------------------------------- schedule
@dataclass
class OracleResult:
    final: np.ndarray
    staleness: list = field(default_factory=list)       # (layer, used, generated)
    dispatch_bytes: int = 0
    combine_bytes: int = 0
    peak_buffer_bytes: int = 0
    active_pairs: int = 0
    total_pairs: int = 0
    per_step_active: list = field(default_factory=list)
    per_step_total: list = field(default_factory=list)
    inputs: list = field(default_factory=list)          # [step][layer] u
    routes: list = field(default_factory=list)          # [step][layer] Route
    masks: list = field(default_factory=list)           # [step][layer] active

    def histogram(self) -> dict:
        out = {}
        for _, used, gen in self.staleness:
            out[used - gen] = out.get(used - gen, 0) + 1
        return dict(sorted(out.items()))


class DivergedAt(Exception):
    def __init__(self, step):
        super().__init__(f"non-finite sample values at step {step}")
        self.step = step


def run_schedule(g: Geometry, params: list, x0: np.ndarray, strategy: str,
                 policy: Policy, devices: int, seed: int, *, record=False,
                 layer_limit=None, step_limit=None, forced_ids=None) -> OracleResult:
    """Restatement of ScheduleRunner (schedules.py:142-490).

    Per step, per layer: mixing block, gate, then a synchronous, displaced or
    interweaved MoE stage; after the stack, x <- x - eta*h.  Stage choice
    follows ``_stage_is_sync`` (schedules.py:406-416); the interweaved stage
    keeps one pending dispatch and one combine slot per layer
    (schedules.py:372-402); the displaced stage keeps a dispatch and a combine
    slot per layer (347-370).  ``layer_limit``/``step_limit`` bound the work
    for CPU timing samples only. ``forced_ids[step][layer]`` teacher-forces the
    routing decisions (e.g. to the ids a device run produced) so schedule
    accounting and latents can be compared without route-flip amplification.
    """
    if policy.cond_strategy == COND_RANDOM and policy.cond_seed is None:   # schedules.py:158-159
        policy = Policy(**{**policy.__dict__, "cond_seed": seed})
    L = g.num_layers if layer_limit is None else layer_limit
    steps = g.num_steps if step_limit is None else step_limit
    n, k, h = g.total_rows, g.top_k, g.hidden_dim
    expert_dev, home = placement(g.num_experts, devices, n)
    sync_set = sync_layer_set(policy.sync_strategy, g.num_layers, policy.explicit_layers)
    cache = CadenceCache(g.num_layers, n, k, h) if policy.cond_strategy != COND_OFF else None
    res = OracleResult(final=None)
    slot_bytes = n * h * 2
    occupied = set()
    dispatch_slot = [None] * g.num_layers      # displaced only
    combine_slot = [None] * g.num_layers       # (rows, gates, generated_step)
    pending = None                             # interweaved only

    def decide(layer, step, route, force):
        if cache is None:
            return np.ones((n, k), bool), np.zeros((n, k), bool)
        return cache.decide(layer, step, route.ids, policy, force)

    def compute(payload):
        layer, u, route, active, write, gen = payload
        rows = expert_rows(params[layer], u, route, active)
        gates = route.gates
        if cache is not None:
            rows, gates = cache.assemble(layer, rows, route, active, write)
        res.combine_bytes += remote_pair_bytes(route.ids, active, expert_dev, home, h)
        return rows, gates, gen

    def store(kind, layer, value):
        occupied.add((kind, layer))
        res.peak_buffer_bytes = max(res.peak_buffer_bytes, len(occupied) * slot_bytes)
        (dispatch_slot if kind == "d" else combine_slot)[layer] = value

    x = x0
    for step in range(steps):
        act_here = tot_here = 0
        u_rec, r_rec, m_rec = [], [], []
        hcur = x
        for layer in range(L):
            p = params[layer]
            u = mixing_block(p, hcur)
            if forced_ids is None:
                route = route_tokens(u, p.w_gate, k)
            else:
                route = forced_route(u, p.w_gate, forced_ids[step][layer])
            if strategy == SYNC or sync_step(step, policy.warmup, policy.period) \
                    or layer in sync_set:
                is_sync = True
            elif strategy == DISPLACED:
                is_sync = dispatch_slot[layer] is None or combine_slot[layer] is None
            else:
                is_sync = combine_slot[layer] is None
            if is_sync:
                if pending is not None:                                    # schedules.py:435
                    prev, pending = pending, None
                    store("c", prev[0], compute(prev))
                active, write = decide(layer, step, route, True)
                payload = (layer, u, route, active, write, step)
                res.dispatch_bytes += remote_pair_bytes(route.ids, active, expert_dev, home, h)
                consumed = compute(payload)
                if strategy == DISPLACED:
                    store("d", layer, payload)
                    store("c", layer, consumed)
                elif strategy == INTERWEAVED:
                    store("c", layer, consumed)
            elif strategy == DISPLACED:
                active, write = decide(layer, step, route, False)
                res.dispatch_bytes += remote_pair_bytes(route.ids, active, expert_dev, home, h)
                old = dispatch_slot[layer]
                store("d", layer, (layer, u, route, active, write, step))
                fresh = compute(old)
                consumed = combine_slot[layer]
                store("c", layer, fresh)
            else:
                active, write = decide(layer, step, route, False)
                res.dispatch_bytes += remote_pair_bytes(route.ids, active, expert_dev, home, h)
                prev, pending = pending, (layer, u, route, active, write, step)
                if prev is not None:
                    store("c", prev[0], compute(prev))
                consumed = combine_slot[layer]
            act_here += int(np.count_nonzero(active))
            tot_here += active.size
            rows, gates, gen = consumed
            shared = shared_sum(p, u)
            hcur = u + weighted_combine(rows, shared, gates)
            res.staleness.append((layer, step, gen))
            if record:
                u_rec.append(u)
                r_rec.append(route)
                m_rec.append(active)
        if pending is not None:                                            # schedules.py:443
            prev, pending = pending, None
            store("c", prev[0], compute(prev))
        x = x - g.step_size * hcur                                         # model.py:301-305
        if not np.isfinite(x).all():
            raise DivergedAt(step)
        res.per_step_active.append(act_here)
        res.per_step_total.append(tot_here)
        res.active_pairs += act_here
        res.total_pairs += tot_here
        if record:
            res.inputs.append(u_rec)
            res.routes.append(r_rec)
            res.masks.append(m_rec)
    res.final = x
    return res


def step_similarity(inputs: list, routes: list):
    """Adjacent-step drift (model.py:316-346): per layer, the mean over adjacent
    step pairs of cos(u_s, u_{s+1}) (_cosine, 316-320: 1 if both norms are 0,
    0 if one is) and of the top-1 routing agreement. Returns
    (per_layer_cosine, per_layer_agreement) as fp64 arrays."""
    steps, layers = len(inputs), len(inputs[0])
    cos = np.zeros(layers)
    agree = np.zeros(layers)
    for layer in range(layers):
        c, a = [], []
        for s in range(steps - 1):
            x, y = inputs[s][layer], inputs[s + 1][layer]
            nx, ny = np.linalg.norm(x), np.linalg.norm(y)
            if nx == 0.0 or ny == 0.0:
                c.append(1.0 if nx == ny else 0.0)
            else:
                c.append(float(np.dot(x.ravel(), y.ravel()) / (nx * ny)))
            a.append(float(np.mean(routes[s][layer].ids[:, 0] == routes[s + 1][layer].ids[:, 0])))
        cos[layer] = np.mean(c)
        agree[layer] = np.mean(a)
    return cos, agree


# --------------------------------------------------------------------- presets
# Geometry presets for the BASELINE configs (SURVEY.md §8 preset table). The
# reference only ships h=32/e=64 toys (model.py:93-99); widths are pinned here.
PRESETS = {
    "s2-8e2a": dict(num_layers=12, num_experts=8, num_shared=2, top_k=2,
                    hidden_dim=384, expert_dim=1536, num_tokens=256),
    "xl2-8e2a": dict(num_layers=28, num_experts=8, num_shared=2, top_k=2,
                     hidden_dim=1152, expert_dim=4608, num_tokens=256, step_size=2e-5),
    "g-16e2a": dict(num_layers=40, num_experts=16, num_shared=2, top_k=2,
                    hidden_dim=1664, expert_dim=6656, num_tokens=1024, step_size=2e-6),
}
