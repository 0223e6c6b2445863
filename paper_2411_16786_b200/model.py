"""Model, weights and the per-layer MoE math on the GPU — drop-in for
dicesim.model (/root/reference/pkg/src/dicesim/model.py).

Same names and call signatures as the reference; values are torch CUDA
tensors computed by the sm_100a library (include/dice_b200.h):

* weights are generated on the device from the reference's splitmix64 stream
  (bit-exact fp64, model.py:28-50, 133-162) and stored transposed/padded in the
  layouts the tcgen05 GEMM reads (bf16 operands, fp32 gate);
* the residual stream, gate, softmax and combine are fp32; GEMM operands
  bf16 with fp32 accumulation (SURVEY.md §8 dtype policy).
"""
from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import ops
from .errors import ConfigurationError, ContractError, NumericsError

SPLITMIX_GAMMA = 0x9E3779B97F4A7C15
SPLITMIX_MIX1 = 0xBF58476D1CE4E5B9
SPLITMIX_MIX2 = 0x94D049BB133111EB
_U64 = 0xFFFFFFFFFFFFFFFF
_X0_STREAM_TAG = 0xD1CE0B5E55ED5EED   # model.py:23


@dataclass(frozen=True)
class ModelConfig:
    """Same fields, defaults and validation as model.py:58-90."""
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

    def __post_init__(self):
        if self.num_layers < 1:
            raise ConfigurationError(f"num_layers must be >= 1, got {self.num_layers}")
        if self.num_experts < 1:
            raise ConfigurationError(f"num_experts must be >= 1, got {self.num_experts}")
        if self.num_shared < 0:
            raise ConfigurationError(f"num_shared must be >= 0, got {self.num_shared}")
        if not 1 <= self.top_k <= self.num_experts:
            raise ConfigurationError(
                f"top_k must be in [1, num_experts={self.num_experts}], got {self.top_k}")
        for name in ("hidden_dim", "expert_dim", "num_tokens", "batch", "num_steps"):
            if getattr(self, name) < 1:
                raise ConfigurationError(f"{name} must be >= 1, got {getattr(self, name)}")
        if not (self.step_size > 0 and math.isfinite(self.step_size)):
            raise ConfigurationError(f"step_size must be finite and > 0, got {self.step_size}")
        if self.num_experts > 64:
            raise ConfigurationError("the CUDA path supports up to 64 routed experts")

    @property
    def total_rows(self) -> int:
        return self.num_tokens * self.batch


PRESETS = {
    # reference toys (model.py:93-99)
    "xl-toy": dict(num_layers=28, num_experts=8, num_shared=2, step_size=2e-4),
    "g-toy": dict(num_layers=40, num_experts=16, num_shared=2, step_size=2e-6),
    # BASELINE geometries pinned in SURVEY.md §8 (widths are an external assumption)
    "s2-8e2a": dict(num_layers=12, num_experts=8, num_shared=2, top_k=2, hidden_dim=384,
                    expert_dim=1536, num_tokens=256, batch=4, num_steps=10, step_size=2e-4),
    "xl2-8e2a": dict(num_layers=28, num_experts=8, num_shared=2, top_k=2, hidden_dim=1152,
                     expert_dim=4608, num_tokens=256, batch=32, num_steps=50, step_size=2e-5),
    "g-16e2a": dict(num_layers=40, num_experts=16, num_shared=2, top_k=2, hidden_dim=1664,
                    expert_dim=6656, num_tokens=1024, batch=8, num_steps=50, step_size=2e-6),
}


def preset(name: str, **overrides) -> ModelConfig:
    key = name.lower()
    if key not in PRESETS:
        raise ConfigurationError(f"unknown preset {name!r}; choose from {sorted(PRESETS)}")
    fields = dict(PRESETS[key])
    fields.update(overrides)
    return ModelConfig(**fields)


def mix64(value: int) -> int:
    """Scalar splitmix64 of one key (model.py:39-44) — host-side key derivation."""
    z = (value + SPLITMIX_GAMMA) & _U64
    z = ((z ^ (z >> 30)) * SPLITMIX_MIX1) & _U64
    z = ((z ^ (z >> 27)) * SPLITMIX_MIX2) & _U64
    return z ^ (z >> 31)


def splitmix64(seed: int, count: int, device="cuda") -> torch.Tensor:
    """`count` splitmix64 outputs as an int64 tensor holding the uint64 bits (model.py:28-36)."""
    if count < 0:
        raise ConfigurationError(f"count must be >= 0, got {count}")
    return ops.splitmix_bits(seed, 0, count, device=device)


def _layer_value_count(cfg: ModelConfig) -> int:
    per_expert = cfg.hidden_dim * cfg.expert_dim * 2
    return (cfg.hidden_dim * cfg.hidden_dim + cfg.hidden_dim * cfg.num_experts
            + per_expert * (cfg.num_experts + cfg.num_shared))


@dataclass
class LayerWeights:
    """Device layouts (K-major B operands of C = A @ B^T; pads are zero):
    w_mix_t [hp, hp] bf16 = W_mix^T; w_gate_t [E, hp] f32 = W_gate^T;
    w1_t [E_local*ep, hp] bf16 = stacked W1_e^T; w2_t [E_local*hp, ep] bf16 = stacked W2_e^T;
    ws1_t [S*ep, hp] bf16 = concat_i W1_i^T; ws2_t [hp, S*ep] bf16 = [W2_0; W2_1; ...]^T."""
    w_mix_t: torch.Tensor
    w_gate_t: torch.Tensor
    w1_t: torch.Tensor
    w2_t: torch.Tensor
    ws1_t: torch.Tensor | None
    ws2_t: torch.Tensor | None


@dataclass
class ToyModel:
    config: ModelConfig
    seed: int
    layers: list = field(default_factory=list)
    experts: tuple = (0, 0)      # [first, last) routed experts resident on this device
    hp: int = 0
    ep: int = 0
    device: str = "cuda"

    @property
    def num_local_experts(self) -> int:
        return self.experts[1] - self.experts[0]


def init_model(config: ModelConfig, seed: int, device="cuda", experts=None) -> ToyModel:
    """Generate every weight on the device from its stream offset (model.py:133-162).

    Consumption order per layer: W_mix, W_gate, routed experts (W1, W2),
    shared experts (W1, W2); entries uniform in [-a, a), a = sqrt(1/fan_in).
    ``experts=(first, last)`` materialises only that routed-expert block
    (expert parallelism); stream offsets are unchanged.
    """
    h, e, E, S = config.hidden_dim, config.expert_dim, config.num_experts, config.num_shared
    hp, ep = ops.pad_hidden(h), ops.pad64(e)
    first, last = experts if experts is not None else (0, E)
    if not 0 <= first <= last <= E:
        raise ConfigurationError(f"expert block {experts} outside [0, {E}]")
    El = last - first
    a_h = float(np.sqrt(1.0 / h))
    a_e = float(np.sqrt(1.0 / e))
    bf = torch.bfloat16
    layers = []
    for layer in range(config.num_layers):
        pos = layer * _layer_value_count(config)
        w_mix_t = torch.zeros(hp, hp, dtype=bf, device=device)
        ops.splitmix_fill(w_mix_t, seed, pos, h, h, a_h, transpose=True)
        pos += h * h
        w_gate_t = torch.zeros(E, hp, dtype=torch.float32, device=device)
        ops.splitmix_fill(w_gate_t, seed, pos, h, E, a_h, transpose=True)
        pos += h * E
        w1_t = torch.zeros(max(El, 1) * ep, hp, dtype=bf, device=device)
        w2_t = torch.zeros(max(El, 1) * hp, ep, dtype=bf, device=device)
        for j in range(E):
            if first <= j < last:
                jl = j - first
                ops.splitmix_fill(w1_t[jl * ep:(jl + 1) * ep], seed, pos, h, e, a_h, transpose=True)
                ops.splitmix_fill(w2_t[jl * hp:(jl + 1) * hp], seed, pos + h * e, e, h, a_e,
                                  transpose=True)
            pos += 2 * h * e
        ws1_t = ws2_t = None
        if S > 0:
            ws1_t = torch.zeros(S * ep, hp, dtype=bf, device=device)
            ws2_t = torch.zeros(hp, S * ep, dtype=bf, device=device)
            for i in range(S):
                ops.splitmix_fill(ws1_t[i * ep:(i + 1) * ep], seed, pos, h, e, a_h, transpose=True)
                _fill_columns(ws2_t, i * ep, seed, pos + h * e, e, h, a_e)
                pos += 2 * h * e
        layers.append(LayerWeights(w_mix_t, w_gate_t, w1_t, w2_t, ws1_t, ws2_t))
    return ToyModel(config=config, seed=seed, layers=layers, experts=(first, last), hp=hp, ep=ep,
                    device=str(device))


def _fill_columns(dst, col0, seed, start, rows, cols, a):
    """Write the transposed [cols, rows] stream block into dst[:, col0:col0+rows]."""
    view = dst.view(-1)[col0:]
    # transpose=1 writes out[c*ld + r]; ld = full row stride of dst
    from . import _lib
    _lib.call("dice_splitmix_fill", seed & _U64, start, rows, cols, float(a), 1, 2,
              view.data_ptr(), dst.shape[1], ops._stream())


def model_hash(model: ToyModel) -> str:
    """Identity of the weights. Weights are a pure function of (config, seed,
    expert block), so the hash covers those instead of re-reading ~GBs of HBM
    (the reference hashes the fp64 arrays, model.py:165-178)."""
    d = hashlib.sha256()
    d.update(repr(model.config).encode())
    d.update(f"seed={model.seed};experts={model.experts};layout=bf16-sm100".encode())
    return d.hexdigest()


@dataclass
class ActivationBlock:
    """A token-row matrix plus provenance tags (model.py:189-194). `values` is
    an f32 CUDA tensor [rows, hidden]."""
    values: torch.Tensor
    generated_step: int
    layer: int = -1


@dataclass
class RouteDecision:
    """Top-k routing (model.py:197-206): expert_ids int64 [n, k] (descending
    score, ties to the lower id), gates f32 [n, k], scores f32 [n, E]."""
    expert_ids: torch.Tensor
    gates: torch.Tensor
    scores: torch.Tensor

    @property
    def top_k(self) -> int:
        return self.expert_ids.shape[1]


def sample_x0(config: ModelConfig, seed: int, device="cuda") -> ActivationBlock:
    """x0 uniform in [-1, 1) from the tagged stream, fp32 (model.py:181-186)."""
    x = torch.empty(config.total_rows, config.hidden_dim, dtype=torch.float32, device=device)
    ops.splitmix_fill(x, mix64(seed ^ _X0_STREAM_TAG), 0, config.total_rows, config.hidden_dim,
                      1.0)
    return ActivationBlock(values=x, generated_step=0)


# --------------------------------------------------------------- functional
def _padded(model: ToyModel, values: torch.Tensor, what: str):
    if values.ndim != 2 or values.shape[1] != model.config.hidden_dim:
        raise ContractError(
            f"{what} expects [n, {model.config.hidden_dim}] values, got {tuple(values.shape)}")
    v = values.to(device=model.device, dtype=torch.float32)
    n = v.shape[0]
    u32 = torch.empty(n, model.hp, dtype=torch.float32, device=model.device)
    u16 = torch.empty(n, model.hp, dtype=torch.bfloat16, device=model.device)
    ops.pack_rows(v.contiguous(), model.hp, u32, u16)
    return u32, u16


def gate(model: ToyModel, layer: int, x: ActivationBlock) -> RouteDecision:
    """Softmax routing over experts, top_k slots renormalised (model.py:209-223)."""
    cfg = model.config
    u32, _ = _padded(model, x.values, "gate")
    n, k, E = u32.shape[0], cfg.top_k, cfg.num_experts
    ids = torch.empty(n, k, dtype=torch.int32, device=model.device)
    gates = torch.empty(n, k, dtype=torch.float32, device=model.device)
    scores = torch.empty(n, E, dtype=torch.float32, device=model.device)
    status = torch.empty(4, dtype=torch.int32, device=model.device)
    ops.status_reset(status)
    ops.gate_topk(u32, model.layers[layer].w_gate_t, k, ids, gates, scores, status, 0, layer)
    if int(status[0].item()) != 2 ** 31 - 1:
        raise NumericsError(f"non-finite activations entering gate at layer {layer}")
    return RouteDecision(expert_ids=ids.long(), gates=gates, scores=scores)


def _local_expert(model: ToyModel, expert_id: int) -> int:
    first, last = model.experts
    if not first <= expert_id < last:
        raise ContractError(f"expert {expert_id} is not resident on this device ({model.experts})")
    return expert_id - first


def expert_forward(model: ToyModel, layer: int, expert_id: int, tokens) -> torch.Tensor:
    """gelu(tokens @ W1) @ W2 on the tensor cores (model.py:226-232)."""
    _, t16 = _padded(model, torch.as_tensor(tokens), "expert_forward")
    lw = model.layers[layer]
    j = _local_expert(model, expert_id)
    hp, ep = model.hp, model.ep
    hid = torch.empty(t16.shape[0], ep, dtype=torch.bfloat16, device=model.device)
    out = torch.empty(t16.shape[0], hp, dtype=torch.float32, device=model.device)
    ops.gemm(ops.EPI_GELU_BF16, t16, lw.w1_t[j * ep:(j + 1) * ep], out_bf16=hid)
    ops.gemm(ops.EPI_STORE_F32, hid, lw.w2_t[j * hp:(j + 1) * hp], out_f32=out)
    return out[:, :model.config.hidden_dim]


def shared_forward(model: ToyModel, layer: int, x: ActivationBlock) -> torch.Tensor:
    """Sum of shared-expert MLPs as one concatenated FFN (model.py:235-241):
    sum_i gelu(u W1_i) W2_i = gelu(u [W1_0 .. W1_S]) [W2_0; ..; W2_S]."""
    cfg = model.config
    _, u16 = _padded(model, x.values, "shared_forward")
    n = u16.shape[0]
    out = torch.zeros(n, model.hp, dtype=torch.float32, device=model.device)
    lw = model.layers[layer]
    if cfg.num_shared > 0:
        hid = torch.empty(n, cfg.num_shared * model.ep, dtype=torch.bfloat16, device=model.device)
        ops.gemm(ops.EPI_GELU_BF16, u16, lw.ws1_t, out_bf16=hid)
        ops.gemm(ops.EPI_STORE_F32, hid, lw.ws2_t, out_f32=out)
    return out[:, :cfg.hidden_dim]


def local_block(model: ToyModel, layer: int, x: ActivationBlock) -> ActivationBlock:
    """gelu(x W_mix) + x, fused residual epilogue (model.py:244-252)."""
    x32, x16 = _padded(model, x.values, "local_block")
    out = torch.empty_like(x32)
    ops.gemm(ops.EPI_GELU_RESID, x16, model.layers[layer].w_mix_t, out_f32=out, residual=x32)
    return ActivationBlock(values=out[:, :model.config.hidden_dim], generated_step=x.generated_step,
                           layer=layer)


class _PermuteScratch:
    """Per-shape workspace of the permute kernels (scratch[0] starts at zero)."""
    _cache: dict = {}

    @classmethod
    def get(cls, n, k, E, device):
        key = (n, k, E, str(device))
        if key not in cls._cache:
            cls._cache[key] = torch.zeros(ops.permute_scratch_ints(n, k, E), dtype=torch.int32,
                                          device=device)
        return cls._cache[key]


def routed_rows(model: ToyModel, layer: int, tokens, route: RouteDecision,
                active=None) -> torch.Tensor:
    """[k, n, h] per-slot expert outputs via permute -> grouped tcgen05 FFN ->
    unpermute; inactive pairs stay zero (model.py:255-276)."""
    cfg = model.config
    if model.num_local_experts != cfg.num_experts:
        raise ContractError("routed_rows needs every routed expert resident (use the engine for EP)")
    tokens = torch.as_tensor(tokens)
    n, k = route.expert_ids.shape
    if tokens.shape[0] != n:
        raise ContractError(f"routed_rows: {tokens.shape[0]} token rows vs {n} routed rows")
    _, u16 = _padded(model, tokens, "routed_rows")
    dev = model.device
    E, hp, ep = cfg.num_experts, model.hp, model.ep
    ids = route.expert_ids.to(device=dev, dtype=torch.int32).contiguous()
    gates = route.gates.to(device=dev, dtype=torch.float32).contiguous()
    act = None if active is None else torch.as_tensor(active).to(device=dev, dtype=torch.uint8).contiguous()
    max_rows = ops.permute_max_rows(n, k, E)
    x_perm = torch.empty(max_rows, hp, dtype=torch.bfloat16, device=dev)
    pos = torch.empty(n, k, dtype=torch.int32, device=dev)
    tiles = torch.empty(E + 1, dtype=torch.int32, device=dev)
    counters = torch.zeros(2, dtype=torch.int64, device=dev)
    ops.route_permute(ids, act, u16, x_perm, pos, tiles, counters,
                      _PermuteScratch.get(n, k, E, dev), E)
    hid = torch.empty(max_rows, ep, dtype=torch.bfloat16, device=dev)
    y = torch.empty(max_rows, hp, dtype=torch.bfloat16, device=dev)
    lw = model.layers[layer]
    ops.grouped_ffn(x_perm, lw.w1_t, lw.w2_t, E, tiles, hid, y)
    routed = torch.empty(n, hp, dtype=torch.float32, device=dev)
    rows = torch.empty(k, n, hp, dtype=torch.float32, device=dev)
    ops.cache_assemble(y, pos, act, None, gates, ids, routed, rows_out=rows)
    return rows[:, :, :cfg.hidden_dim]


def combine_outputs(route: RouteDecision, expert_outs, shared_out, scale_route: RouteDecision):
    """shared_out + sum_s scale_route.gates[s] * expert_outs[s] (model.py:279-298)."""
    if expert_outs.shape[0] != route.top_k or expert_outs.shape[0] != scale_route.top_k:
        raise ContractError(
            f"combine_outputs: {expert_outs.shape[0]} slots vs route k={route.top_k}, "
            f"scale k={scale_route.top_k}")
    if expert_outs.shape[1] != shared_out.shape[0]:
        raise ContractError(
            f"combine_outputs: {expert_outs.shape[1]} routed rows vs "
            f"{shared_out.shape[0]} shared rows")
    k, n, h = expert_outs.shape
    dev = shared_out.device
    base = shared_out.to(torch.float32).contiguous()
    rows = expert_outs.to(torch.float32).contiguous()
    # the combine kernel needs a row length that is a multiple of 4
    hp = (h + 3) // 4 * 4
    if hp != h:
        base = torch.nn.functional.pad(base, (0, hp - h))
        rows = torch.nn.functional.pad(rows, (0, hp - h))
    out = torch.empty(n, hp, dtype=torch.float32, device=dev)
    ops.combine(base, rows, scale_route.gates.to(device=dev, dtype=torch.float32).contiguous(), out)
    return out[:, :h]


def denoise_update(x: ActivationBlock, y, eta: float, step: int) -> ActivationBlock:
    """x_{s+1} = x_s - eta * y_s (model.py:301-305)."""
    if tuple(y.shape) != tuple(x.values.shape):
        raise ContractError(f"denoise_update: y shape {tuple(y.shape)} vs x shape {tuple(x.values.shape)}")
    n, h = x.values.shape
    hp = (h + 3) // 4 * 4
    xv = torch.nn.functional.pad(x.values.to(torch.float32), (0, hp - h)).contiguous()
    yv = torch.nn.functional.pad(torch.as_tensor(y, device=xv.device).to(torch.float32), (0, hp - h)).contiguous()
    ops.denoise(xv, None, yv, eta)
    return ActivationBlock(values=xv[:, :h], generated_step=step + 1)


@dataclass
class StepSimilarity:
    """model.py:308-313."""
    per_layer_cosine: object
    per_layer_agreement: object
    mean_cosine: float
    mean_agreement: float


def similarity_from_sums(sums, rows: int) -> StepSimilarity:
    """StepSimilarity from the device sums f64 [layers, steps-1, 4] =
    {a.b, |a|^2, |b|^2, top-1 agreements} of each adjacent step pair
    (_cosine and the agreement mean, model.py:316-346)."""
    sums = np.asarray(sums, dtype=np.float64)
    layers, pairs = sums.shape[:2]
    cos = np.zeros(layers)
    agree = np.zeros(layers)
    for layer in range(layers):
        c_vals, a_vals = [], []
        for s in range(pairs):
            dot, aa, bb, same = sums[layer, s]
            na, nb = float(np.sqrt(aa)), float(np.sqrt(bb))
            if na == 0.0 or nb == 0.0:
                c_vals.append(1.0 if na == nb else 0.0)
            else:
                c_vals.append(float(dot / (na * nb)))
            a_vals.append(float(same) / rows)
        cos[layer] = np.mean(c_vals)
        agree[layer] = np.mean(a_vals)
    return StepSimilarity(per_layer_cosine=cos, per_layer_agreement=agree,
                          mean_cosine=float(np.mean(cos)), mean_agreement=float(np.mean(agree)))


def step_similarity(inputs: list, routes: list) -> StepSimilarity:
    """Adjacent-step cosine of each layer's MoE input and top-1 routing
    agreement (model.py:323-346), reduced on the device
    (dice_step_similarity: fp64 sums in a fixed order, one D2H read).
    inputs[s][l]: [rows, h]; routes[s][l]: RouteDecision."""
    steps = len(inputs)
    if steps < 2:
        raise ContractError("step_similarity needs at least two recorded steps")
    layers = len(inputs[0])
    dev = torch.device("cuda", torch.cuda.current_device())
    rows = int(torch.as_tensor(inputs[0][0]).shape[0])
    sums = torch.empty(layers, steps - 1, 4, dtype=torch.float64, device=dev)
    part = torch.empty(ops.similarity_partial_words(), dtype=torch.float64, device=dev)

    def f32(v):
        return torch.as_tensor(v).to(device=dev, dtype=torch.float32).contiguous()

    def i32(r):
        return torch.as_tensor(r.expert_ids).to(device=dev, dtype=torch.int32).contiguous()

    for layer in range(layers):
        a, ia = f32(inputs[0][layer]), i32(routes[0][layer])
        for s in range(steps - 1):
            b, ib = f32(inputs[s + 1][layer]), i32(routes[s + 1][layer])
            if tuple(b.shape) != tuple(a.shape):
                raise ContractError(f"step_similarity: input shapes {tuple(a.shape)} vs "
                                    f"{tuple(b.shape)}")
            ops.step_similarity(a, b, a.shape[1], ia, ib, sums[layer, s], part)
            a, ia = b, ib
    return similarity_from_sums(sums.cpu().numpy(), rows)
