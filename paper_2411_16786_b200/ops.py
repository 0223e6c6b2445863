"""Tensor-level wrappers over the C-ABI (torch CUDA tensors in, CUDA kernels out).

torch is used only for device memory and the current stream; every value is
computed by the sm_100a library. Shapes use padded feature dims (multiples of
64, zero padding) as include/dice_b200.h specifies.
"""
from __future__ import annotations

import torch

from . import _lib
from .errors import ContractError

EPI_STORE_BF16, EPI_GELU_BF16, EPI_STORE_F32, EPI_GELU_RESID = range(4)
COND_CODES = {"off": 0, "low_score": 1, "high_score": 2, "random": 3}


def pad64(x: int) -> int:
    return (x + 63) // 64 * 64


def pad_hidden(h: int) -> int:
    """Padded hidden width of the device layouts: a multiple of 64, raised to a
    multiple of 256 when that costs <= 10 % and the 64-multiple would leave the
    N = hidden GEMMs on 128-wide tiles (e.g. the G preset, 1664 -> 1792). Pads
    are zero in every weight and activation, so values are unchanged."""
    hp = pad64(h)
    if hp % 192 == 0 or hp % 256 == 0:
        return hp
    h256 = (h + 255) // 256 * 256
    return h256 if h256 <= 1.1 * hp else hp


def _ptr(t):
    return None if t is None else t.data_ptr()


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _need(t, dtype, what):
    if t is None:
        return
    if not t.is_cuda:
        raise ContractError(f"{what}: expected a CUDA tensor")
    if t.dtype != dtype:
        raise ContractError(f"{what}: expected {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ContractError(f"{what}: expected a contiguous tensor")


class DeviceEvent:
    """CUDA event usable inside CUDA-graph capture (external event node)."""

    def __init__(self):
        import ctypes
        h = ctypes.c_void_p()
        _lib.call("dice_event_create", ctypes.byref(h))
        self.handle = h

    def record(self):
        _lib.call("dice_event_record", self.handle, _stream())

    def elapsed_ms(self, end: "DeviceEvent") -> float:
        import ctypes
        ms = ctypes.c_float()
        _lib.call("dice_event_elapsed_ms", self.handle, end.handle, ctypes.byref(ms))
        return float(ms.value)

    def __del__(self):
        try:
            _lib.load().dice_event_destroy(self.handle)
        except Exception:
            pass


def status_reset(status):
    _lib.call("dice_status_reset", _ptr(status), _stream())


def splitmix_fill(out, seed, start, rows, cols, halfwidth, transpose=False):
    """Fill `out` (f64/f32/bf16, row stride out.shape[-1]) from the splitmix64 stream."""
    code = {torch.float64: 0, torch.float32: 1, torch.bfloat16: 2}[out.dtype]
    _lib.call("dice_splitmix_fill", seed & 0xFFFFFFFFFFFFFFFF, start, rows, cols,
              float(halfwidth), int(transpose), code, _ptr(out), out.shape[-1], _stream())


def splitmix_bits(seed, start, count, device="cuda"):
    out = torch.empty(count, dtype=torch.int64, device=device)
    _lib.call("dice_splitmix_bits", seed & 0xFFFFFFFFFFFFFFFF, start, count, _ptr(out), _stream())
    return out


def _decide_args(decide):
    if decide is None:
        return (0, 0, 1, 0, 0, 0, None, None, None, None, None, None)
    (force, R, strat, strict, key, last, primed, reduced, cached, active, write) = decide
    return (1, int(force), R, strat, int(strict), key & 0xFFFFFFFFFFFFFFFF, _ptr(last),
            _ptr(primed), _ptr(reduced), _ptr(cached), _ptr(active), _ptr(write))


def gate_topk(u32, w_gate_t, k, ids, gates, scores=None, status=None, step=0, layer=0,
              decide=None):
    """Fused gate (softmax + stable top-k); ``decide`` = TokenCache.decide_args(...)
    also runs the conditional-communication decision in the same kernel."""
    n, hp = u32.shape
    E = w_gate_t.shape[0]
    _need(u32, torch.float32, "gate u")
    if decide is None:
        _lib.call("dice_gate_topk", _ptr(u32), _ptr(w_gate_t), n, hp, E, k, _ptr(ids),
                  _ptr(gates), _ptr(scores), _ptr(status), step, layer, _stream())
        return
    (force, R, strat, strict, key, last, primed, reduced, cached, active, write) = decide
    _lib.call("dice_gate_topk_decide", _ptr(u32), _ptr(w_gate_t), n, hp, E, k, _ptr(ids),
              _ptr(gates), _ptr(scores), _ptr(status), step, layer, int(force), R, strat,
              int(strict), key & 0xFFFFFFFFFFFFFFFF, _ptr(last), _ptr(primed), _ptr(reduced),
              _ptr(cached), _ptr(active), _ptr(write), _stream())


def route_state_words(n):
    return int(_lib.load().dice_gate_route_state_words(n))


def gate_route(u32, w_gate_t, k, ids, gates, x_perm, cap, pos, row_pair, tile_offsets, counters,
               state, scores=None, status=None, step=0, layer=0, decide=None, devices=1,
               rows_total=None):
    """Gate + conditional-communication decision + token permute in one launch
    (E = 8 or 16): x_perm bf16 [E*cap, hp], expert e's rows from e*cap (dice_gate_route)."""
    n, hp = u32.shape
    E = w_gate_t.shape[0]
    _need(u32, torch.float32, "gate u")
    _need(x_perm, torch.bfloat16, "x_perm")
    _need(state, torch.int64, "route state")
    if x_perm.shape[0] < E * cap or state.numel() < route_state_words(n):
        raise ContractError("gate_route: x_perm / route state too small")
    _lib.call("dice_gate_route", _ptr(u32), _ptr(w_gate_t), n, hp, E, k, _ptr(ids), _ptr(gates),
              _ptr(scores), _ptr(status), step, layer, *_decide_args(decide), _ptr(x_perm), cap,
              _ptr(pos), _ptr(row_pair), _ptr(tile_offsets), _ptr(counters), devices,
              n if rows_total is None else rows_total, _ptr(state), _stream())


def cond_decide(ids, step, force, refresh_interval, strategy, strict, random_key, last, primed,
                reduced, cached_ids, active, write):
    n, k = ids.shape
    _lib.call("dice_cond_decide", _ptr(ids), n, k, step, int(force), refresh_interval,
              COND_CODES[strategy], int(strict), random_key & 0xFFFFFFFFFFFFFFFF, _ptr(last),
              _ptr(primed), _ptr(reduced), _ptr(cached_ids), _ptr(active), _ptr(write), _stream())


def permute_max_rows(n, k, E):
    return int(_lib.load().dice_permute_max_rows(n, k, E))


def permute_scratch_ints(n, k, E):
    return int(_lib.load().dice_permute_scratch_ints(n, k, E))


def route_permute(ids, active, u16, x_perm, pos, tile_offsets, counters, scratch, E,
                  devices=1, row0=0, rows_total=None, row_pair=None):
    """row_pair (int32 [max_rows], optional): permuted row -> pair index t*k+s
    (-1 on padding rows), for the expert GEMM2's pair-row stores."""
    n, k = ids.shape
    hp = u16.shape[1]
    _lib.call("dice_route_permute", _ptr(ids), _ptr(active), n, k, E, _ptr(u16), hp,
              _ptr(x_perm), x_perm.shape[0], _ptr(pos), _ptr(tile_offsets), _ptr(counters),
              devices, row0, n if rows_total is None else rows_total, _ptr(scratch),
              _ptr(row_pair), _stream())


def grouped_ffn(x_perm, w1_t, w2_t, E, tile_offsets, hbuf, y):
    max_rows, hp = x_perm.shape
    ep = hbuf.shape[1]
    _lib.call("dice_grouped_ffn", _ptr(x_perm), max_rows, _ptr(w1_t), _ptr(w2_t), E, hp, ep,
              _ptr(tile_offsets), _ptr(hbuf), _ptr(y), _stream())


def expert_gemm1_with_shared(x_perm, w1_t, E, tile_offsets, hbuf, u16, ws1_t, hsh,
                             group_stride=0):
    """Grouped expert GEMM1 (+GELU) and the shared experts' GEMM1 (+GELU) in
    one persistent launch (dice_expert_gemm1_with_dense). group_stride > 0:
    expert e's rows of x_perm start at e * group_stride (dice_gate_route)."""
    max_rows, ep = hbuf.shape
    hp = x_perm.shape[1]
    _lib.call("dice_expert_gemm1_with_dense", _ptr(x_perm), max_rows, group_stride, _ptr(w1_t), E,
              hp, ep, _ptr(tile_offsets), _ptr(hbuf), _ptr(u16), u16.shape[0], _ptr(ws1_t),
              ws1_t.shape[0], _ptr(hsh), _stream())


def expert_gemm2(hbuf, w2_t, E, tile_offsets, y):
    max_rows, ep = hbuf.shape
    hp = y.shape[1]
    _lib.call("dice_expert_gemm2", _ptr(hbuf), max_rows, _ptr(w2_t), E, hp, ep, _ptr(tile_offsets),
              _ptr(y), _stream())


def expert_gemm2_pairs(hbuf, w2_t, E, tile_offsets, row_pair, gates, ids, pair_rows,
                       cache_gates=None, cache_ids=None, pair_group_stride=0):
    """Expert GEMM2 whose epilogue stores each row of pair p = t*k + s into
    pair_rows[s, t] (bf16 [k, n, hp]) and persists the pair's gate / expert id
    (dice_expert_gemm2_pairs)."""
    max_rows, ep = hbuf.shape
    n, k = gates.shape
    hp = pair_rows.shape[-1]
    _need(pair_rows, torch.bfloat16, "pair rows")
    if tuple(pair_rows.shape) != (k, n, hp):
        raise ContractError(f"pair rows {tuple(pair_rows.shape)} != {(k, n, hp)}")
    _lib.call("dice_expert_gemm2_pairs", _ptr(hbuf), max_rows, _ptr(w2_t), E, hp, ep,
              _ptr(tile_offsets), _ptr(row_pair), pair_group_stride, _ptr(gates), _ptr(ids), k, n,
              _ptr(pair_rows), _ptr(cache_gates), _ptr(cache_ids), _stream())


def gemm_consume(A, B, residual, pair_rows, pair_gates, out_f32, out_bf16=None):
    """out = residual + ((A @ B^T + g_0 row_0) + g_1 row_1 ...): the shared-expert
    GEMM2 with the layer's consume fused (dice_gemm_consume)."""
    _need(A, torch.bfloat16, "gemm A")
    _need(B, torch.bfloat16, "gemm B")
    M, K = A.shape
    N = B.shape[0]
    k = pair_gates.shape[1]
    if B.shape[1] != K or tuple(pair_rows.shape) != (k, M, N):
        raise ContractError(f"gemm_consume: A {tuple(A.shape)} B {tuple(B.shape)} "
                            f"rows {tuple(pair_rows.shape)}")
    _lib.call("dice_gemm_consume", _ptr(A), M, _ptr(B), N, K, _ptr(residual), residual.shape[-1],
              _ptr(pair_rows), _ptr(pair_gates), k, _ptr(out_f32), out_f32.shape[-1],
              _ptr(out_bf16), 0 if out_bf16 is None else out_bf16.shape[-1], _stream())


def consume_rows(residual, pair_rows, pair_gates, out_f32, out_bf16=None):
    """out = residual + ((0 + g_0 row_0) + ...) (no shared experts)."""
    n, hp = residual.shape
    k = pair_gates.shape[1]
    _lib.call("dice_consume_rows", _ptr(residual), _ptr(pair_rows), _ptr(pair_gates), n, k, hp,
              _ptr(out_f32), _ptr(out_bf16), _stream())


def cache_assemble(y, pos, active, write, gates, ids, routed, cache_rows=None, cache_gates=None,
                   cache_ids=None, rows_out=None, gates_out=None):
    n, k = pos.shape
    hp = routed.shape[1]
    _lib.call("dice_cache_assemble", _ptr(y), _ptr(pos), _ptr(active), _ptr(write), _ptr(gates),
              _ptr(ids), n, k, hp, _ptr(cache_rows), _ptr(cache_gates), _ptr(cache_ids),
              _ptr(routed), _ptr(rows_out), _ptr(gates_out), _stream())


def gemm(epi, A, B, out_f32=None, out_bf16=None, residual=None):
    """C[M, N] = A[M, K] @ B[N, K]^T (bf16 operands, fp32 accumulate) + fused epilogue."""
    _need(A, torch.bfloat16, "gemm A")
    _need(B, torch.bfloat16, "gemm B")
    M, K = A.shape
    N = B.shape[0]
    if B.shape[1] != K:
        raise ContractError(f"gemm: A {tuple(A.shape)} vs B {tuple(B.shape)}")
    ld = lambda t: 0 if t is None else t.shape[-1]
    _lib.call("dice_gemm", epi, _ptr(A), M, _ptr(B), N, K, _ptr(out_f32), ld(out_f32),
              _ptr(out_bf16), ld(out_bf16), _ptr(residual), ld(residual), _stream())


def combine(base, rows, gates, out, residual=None, out_bf16=None):
    n, hp = base.shape
    k = gates.shape[1]
    _lib.call("dice_combine", _ptr(base), _ptr(rows), _ptr(gates), _ptr(residual), n, k, hp,
              _ptr(out), _ptr(out_bf16), _stream())


def denoise(x32, x16, y, eta, status=None, step=0):
    n, hp = x32.shape
    _lib.call("dice_denoise", _ptr(x32), _ptr(x16), _ptr(y), float(eta), n, hp, _ptr(status),
              step, _stream())


def pack_rows(src, hp, out32=None, out16=None):
    n, cols = src.shape
    _need(src, torch.float32, "pack_rows src")
    _lib.call("dice_pack_rows", _ptr(src), n, cols, src.stride(0), hp, _ptr(out32), _ptr(out16),
              _stream())


def similarity_partial_words():
    return int(_lib.load().dice_similarity_partial_words())


def step_similarity(prev, cur, cols, prev_top, cur_ids, out, partials, roll=False):
    """out f64 [4] = {a.b, |a|^2, |b|^2, #rows with equal top-1} of prev / cur
    (first ``cols`` columns); roll: then prev <- cur, prev_top <- cur's top-1.
    prev_top: int32 [n] or the [n, k] ids of prev (its column 0 is read)."""
    n = cur.shape[0]
    _need(cur, torch.float32, "step_similarity cur")
    _need(cur_ids, torch.int32, "step_similarity ids")
    _need(out, torch.float64, "step_similarity out")
    if prev.dtype != torch.float32 or prev.stride(1) != 1 or cur.stride(1) != 1:
        raise ContractError("step_similarity: f32 row-major inputs expected")
    if prev_top.dtype != torch.int32:
        raise ContractError("step_similarity: int32 top-1 ids expected")
    top_stride = prev_top.stride(0)
    _lib.call("dice_step_similarity", _ptr(prev), _ptr(cur), n, int(cols), prev.stride(0),
              cur.stride(0), _ptr(prev_top), top_stride, _ptr(cur_ids), cur_ids.shape[1],
              int(bool(roll)), _ptr(partials), _ptr(out), _stream())
