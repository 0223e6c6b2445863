// Memory-bound kernels of the DICE MoE layer (sm_100a) and the C-ABI entry
// points declared in include/dice_b200.h. The dense contractions live in
// dice_gemm.cu (tcgen05 / TMEM / TMA).
#include <climits>
#include <cstdlib>
#include <cstdint>

#include "dice_gemm.h"
#include "dice_ptx.cuh"

namespace dice {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;  // model.py:17
constexpr uint64_t kMul1 = 0xBF58476D1CE4E5B9ull;   // model.py:18
constexpr uint64_t kMul2 = 0x94D049BB133111EBull;   // model.py:19

__device__ __forceinline__ uint64_t splitmix_at(uint64_t seed, uint64_t counter) {
  uint64_t z = seed + counter * kGamma;
  z = (z ^ (z >> 30)) * kMul1;
  z = (z ^ (z >> 27)) * kMul2;
  return z ^ (z >> 31);
}

__device__ __forceinline__ void record_nonfinite(int32_t* status, int step, int layer) {
  if (status == nullptr) return;
  const int prev = atomicMin(&status[0], step);
  if (prev > step) atomicExch(&status[1], layer);
}

__device__ __forceinline__ float bf16_bits_to_f32(uint16_t b) {
  return __uint_as_float(static_cast<uint32_t>(b) << 16);
}

// ------------------------------------------------------------------ status
__global__ void status_reset_kernel(int32_t* s) {
  pdl_enter();
  s[0] = INT_MAX;
  s[1] = -1;
  s[2] = 0;
  s[3] = 0;
}

// ----------------------------------------------------------- splitmix fill
// Element (r, c) of the logical row-major [rows, cols] stream block is output
// start + r*cols + c, i.e. counter start + r*cols + c + 1 (model.py:32-33).
// Value = a * (2 * ((bits >> 11) * 2^-53) - 1) in fp64 (model.py:47-50).
__global__ void splitmix_fill_kernel(uint64_t seed, uint64_t start, int64_t rows, int64_t cols,
                                     double a, int transpose, int out_dtype, void* out,
                                     int64_t ld) {
  pdl_enter();
  const int64_t total = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r, c, o;
    if (transpose) { c = i / rows; r = i - c * rows; o = c * ld + r; }
    else { r = i / cols; c = i - r * cols; o = r * ld + c; }
    const uint64_t bits = splitmix_at(seed, start + (uint64_t)(r * cols + c) + 1);
    const double unit = __dmul_rn((double)(bits >> 11), 1.1102230246251565e-16);  // 2^-53
    const double v = __dmul_rn(a, __dsub_rn(__dmul_rn(2.0, unit), 1.0));
    if (out_dtype == 0) {
      static_cast<double*>(out)[o] = v;
    } else if (out_dtype == 1) {
      static_cast<float*>(out)[o] = __double2float_rn(v);
    } else {
      static_cast<__nv_bfloat16*>(out)[o] = __float2bfloat16_rn(__double2float_rn(v));
    }
  }
}

__global__ void splitmix_bits_kernel(uint64_t seed, uint64_t start, int64_t count, uint64_t* out) {
  pdl_enter();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = splitmix_at(seed, start + (uint64_t)i + 1);
}

// -------------------------------------------------------------------- gate
// One warp per token row. W_gate^T staged in shared memory; fp32 dot products
// reduced with butterfly shuffles; softmax; stable top-k by (score desc, id asc)
// (model.py:215-222).
template <int EMAX>
__device__ __forceinline__ void gate_finish(float (&acc)[EMAX], int E, int k, int64_t t, int lane,
                                            int32_t* __restrict__ ids, float* __restrict__ gates,
                                            float* __restrict__ scores) {
#pragma unroll
  for (int e = 0; e < EMAX; ++e) {
    if (e < E) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], o);
    }
  }
  // softmax over the E logits (model.py:216-218)
  float mx = acc[0];
#pragma unroll
  for (int e = 1; e < EMAX; ++e) if (e < E) mx = fmaxf(mx, acc[e]);
  float sum = 0.f;
#pragma unroll
  for (int e = 0; e < EMAX; ++e) if (e < E) { acc[e] = expf(acc[e] - mx); sum += acc[e]; }
#pragma unroll
  for (int e = 0; e < EMAX; ++e) if (e < E) acc[e] = acc[e] / sum;
  if (scores != nullptr) {
#pragma unroll
    for (int e = 0; e < EMAX; ++e) if (e < E && (e & 31) == lane) scores[t * E + e] = acc[e];
  }
  if (lane == 0) {
    // stable top-k on scores: strictly greater wins, so ties keep the lower id
    uint64_t taken = 0;
    int pick[EMAX];
    float pv[EMAX];
    float psum = 0.f;
    for (int j = 0; j < k; ++j) {
      int best = -1;
      float bv = 0.f;
#pragma unroll
      for (int e = 0; e < EMAX; ++e) {
        if (e < E && !((taken >> e) & 1ull) && (best < 0 || acc[e] > bv)) { best = e; bv = acc[e]; }
      }
      taken |= 1ull << best;
      pick[j] = best;
      pv[j] = bv;
      psum += bv;
    }
    for (int j = 0; j < k; ++j) {
      ids[t * k + j] = pick[j];
      gates[t * k + j] = pv[j] / psum;
    }
  }
}

// One warp per pair of token rows (W_gate^T reads from shared memory are
// shared by both rows). fp32 dot products reduced with butterfly shuffles,
// softmax, stable top-k by (score desc, id asc) (model.py:215-222).
template <int EMAX>
__global__ void __launch_bounds__(512) gate_topk_kernel(
    const float* __restrict__ u, const float* __restrict__ wt, int64_t n, int hp, int E, int k,
    int32_t* __restrict__ ids, float* __restrict__ gates, float* __restrict__ scores,
    int32_t* status, int step, int layer) {
  pdl_enter();
  extern __shared__ float sw[];  // [E, hp]
  {
    const float4* src = reinterpret_cast<const float4*>(wt);
    float4* dst = reinterpret_cast<float4*>(sw);
    for (int i = threadIdx.x; i < E * hp / 4; i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  const int64_t pairs = (n + 1) / 2;
  for (int64_t q = blockIdx.x * (int64_t)warps + (threadIdx.x >> 5); q < pairs;
       q += (int64_t)gridDim.x * warps) {
    const int64_t t0 = 2 * q, t1 = 2 * q + 1;
    const bool has1 = t1 < n;
    float a0[EMAX], a1[EMAX];
#pragma unroll
    for (int e = 0; e < EMAX; ++e) { a0[e] = 0.f; a1[e] = 0.f; }
    bool finite = true;
    const float* r0 = u + t0 * hp;
    const float* r1 = u + (has1 ? t1 : t0) * hp;
    constexpr int CH = 4;  // 128-column strips per batch: 2*CH 16-byte loads in flight per lane
    for (int base = 0; base < hp; base += 128 * CH) {
      float4 xs[CH], ys[CH];
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        const int c = base + 128 * j + lane * 4;
        if (c < hp) {
          xs[j] = *reinterpret_cast<const float4*>(r0 + c);
          ys[j] = *reinterpret_cast<const float4*>(r1 + c);
        } else {
          xs[j] = make_float4(0.f, 0.f, 0.f, 0.f);
          ys[j] = xs[j];
        }
      }
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        const int c = base + 128 * j + lane * 4;
        if (c >= hp) break;
        const float4 x = xs[j], y = ys[j];
        finite &= isfinite(x.x) && isfinite(x.y) && isfinite(x.z) && isfinite(x.w);
        finite &= isfinite(y.x) && isfinite(y.y) && isfinite(y.z) && isfinite(y.w);
#pragma unroll
        for (int e = 0; e < EMAX; ++e) {
          if (e < E) {
            const float4 w = *reinterpret_cast<const float4*>(sw + e * hp + c);
            a0[e] = fmaf(x.x, w.x, a0[e]); a0[e] = fmaf(x.y, w.y, a0[e]);
            a0[e] = fmaf(x.z, w.z, a0[e]); a0[e] = fmaf(x.w, w.w, a0[e]);
            a1[e] = fmaf(y.x, w.x, a1[e]); a1[e] = fmaf(y.y, w.y, a1[e]);
            a1[e] = fmaf(y.z, w.z, a1[e]); a1[e] = fmaf(y.w, w.w, a1[e]);
          }
        }
      }
    }
    finite = __all_sync(0xffffffffu, finite);
    if (!finite && lane == 0) record_nonfinite(status, step, layer);
    gate_finish<EMAX>(a0, E, k, t0, lane, ids, gates, scores);
    if (has1) gate_finish<EMAX>(a1, E, k, t1, lane, ids, gates, scores);
  }
}

// Fast gate for E in {8, 16}: two token rows per warp; the 2E per-lane
// partial dot products are reduced with a transpose-reduce (each butterfly
// level exchanges half of the remaining values), leaving lane L with the full
// logit of (row L>>4, expert ...). Softmax and the stable top-k ranking
// (score desc, id asc; model.py:216-222) are then done lane-parallel within
// each row's 16-lane group.
template <int N>
__device__ __forceinline__ void tr_level(float (&a)[32], int lane, int off) {
  const bool upper = (lane & off) != 0;
#pragma unroll
  for (int j = 0; j < N / 2; ++j) {
    const float send = upper ? a[j] : a[j + N / 2];
    const float keep = upper ? a[j + N / 2] : a[j];
    a[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
  }
}

// ------------------------------------------------------------ cond decide
// Per token (policies.py:159-186): due = force | !primed | (step - last) >= R;
// due tokens redraw the reduced-slot subset (policies.py:118-139) and reset the
// cadence; active = !reduced | due; write = reduced & due; strict adds pairs
// whose expert moved since the cached refresh.
struct DecideArgs {
  int on, step, force, R, strategy, strict;
  uint64_t key;
  int32_t* last;
  uint8_t* primed;
  uint8_t* reduced;
  const int32_t* cached_ids;
  uint8_t* active;
  uint8_t* write;
};

// Token permute fused into the router launch (single-GPU engine, E = 8): one
// block = 32 tokens. After the gate and the conditional-communication
// decision, the block's active pairs are grouped by expert (warp match ranks
// in pair order t*k+s, routed_rows' grouping, model.py:263-275, up to the
// within-expert order, which changes no value), the per-expert offsets of the
// earlier blocks are the sums of the blocks' published
// counts, and the block copies its tokens' bf16 rows (rounded from the fp32 u
// it already holds for the gate, the same rounding as the local GEMM's bf16
// output) straight to their permuted positions. Expert e's rows live in a
// fixed-capacity region [e*cap, (e+1)*cap) (cap >= tokens), so no position
// depends on another expert's total; the last block writes the 256-row tile
// prefix and marks the padding rows of every region. Counters: active pairs
// and remote pairs of the byte plan (cluster.py:75-90).
constexpr int kRowTileR = 256;
#ifndef DICE_ROUTER_WPB
#define DICE_ROUTER_WPB 8
#endif
constexpr int kRouterWarps = DICE_ROUTER_WPB;   // warps per router block   // expert regions padded to the CTA-pair GEMM's 256-row tile

struct RouteArgs {
  uint16_t* x_perm;             // [E * cap, hp] bf16; null: gate only
  int64_t cap;                  // rows per expert region (multiple of 256)
  int32_t* pos;                 // [n, k] row of each pair, -1 inactive
  int32_t* row_pair;            // [E * cap] pair of each row, -1 on padding rows
  int32_t* tile_offsets;        // [E + 1] 256-row tile prefix
  long long* counters;          // [2] (+=) active pairs, remote pairs
  int devices;
  int64_t rows_total;
  unsigned* state;              // [9]: finished-block ticket, per-expert row counters
};

// Token rows are read once: keep them out of L1 so W_gate (re-read by every
// warp through L1) stays resident next to the routing launch's smem staging.
__device__ __forceinline__ float4 ldg_stream_f4(const float* p) {
  float4 v;
  asm("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}

__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// TokenCache.decide for token t (policies.py:159-186): cadence, mask redraw,
// active / write masks (strict: also refresh reduced pairs whose expert changed)
__device__ __forceinline__ void decide_token(int64_t t, int k, const int32_t* ids,
                                             const DecideArgs& d) {
  const int step = d.step, strategy = d.strategy;
  int32_t* last = d.last;
  uint8_t* primed = d.primed;
  uint8_t* reduced = d.reduced;
  uint8_t* active = d.active;
  uint8_t* write = d.write;
  {
    if (strategy == DICE_COND_OFF) {
      for (int s = 0; s < k; ++s) { active[t * k + s] = 1; write[t * k + s] = 0; }
      return;
    }
    const int force = d.force, R = d.R, strict = d.strict;
    const uint64_t key = d.key;
    const int32_t* cached_ids = d.cached_ids;
    const bool due = force || !primed[t] || (step - last[t]) >= R;
    if (due) {
      int keep = -1;
      if (strategy == DICE_COND_RANDOM) keep = (int)(splitmix_at(key, (uint64_t)t + 1) % (uint64_t)k);
      for (int s = 0; s < k; ++s) {
        bool red;
        if (strategy == DICE_COND_LOW_SCORE) red = s >= 1;
        else if (strategy == DICE_COND_HIGH_SCORE) red = s == 0;
        else red = s != keep;
        reduced[t * k + s] = red;
      }
      last[t] = step;
      primed[t] = 1;
    }
    for (int s = 0; s < k; ++s) {
      const bool red = reduced[t * k + s] != 0;
      bool a = !red || due;
      bool w = red && due;
      if (strict && red && !due && ids[t * k + s] != cached_ids[t * k + s]) { a = true; w = true; }
      active[t * k + s] = a;
      write[t * k + s] = w;
    }
  }
}

__global__ void cond_decide_kernel(const int32_t* __restrict__ ids, int64_t n, int k,
                                   const DecideArgs d) {
  pdl_enter();
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    decide_token(t, k, ids, d);
}

// Router, warp per RPW = 32 / E rows (E = 8: four rows, E = 16: two). Each
// W_gate float4 (4 columns of one expert) feeds the warp's rows as FFMA2 row
// pairs (E = 8: halving the L1 wavefronts per row), and the RPW x E partial
// logits transpose-reduce to exactly one (row, expert) per lane
// (lane = E row + e). Rows are loaded in CH-chunk batches. One block = 8
// warps = TPB = 8 RPW tokens. With r.x_perm set, the block also permutes its
// pairs (RouteArgs); the bf16 rows are staged in dynamic shared memory.
template <int E, int CH, int WPB>
__global__ void __launch_bounds__(32 * WPB, 2) gate4_topk_kernel(
    const float* __restrict__ u, const float* __restrict__ wt, int64_t n, int hp, int k,
    int32_t* __restrict__ ids, float* __restrict__ gates, float* __restrict__ scores,
    int32_t* status, int step, int layer, const DecideArgs d, const RouteArgs r) {
  static_assert(E == 8 || E == 16, "router handles E = 8 or 16");
  constexpr int RPW = 32 / E;            // rows per warp
  constexpr int NP = RPW / 2;            // FFMA2 row pairs per warp
  constexpr int TPB = WPB * RPW;         // tokens per block
  extern __shared__ __align__(16) uint16_t s_rows[];   // [TPB, hp] bf16 (routing only)
  __shared__ int s_wcnt[WPB][E];     // per (warp, expert): count, then exclusive prefix
  __shared__ int s_base[E];
  __shared__ int s_tot[E];
  __shared__ int s_fin;
  __shared__ int s_pos[TPB * E];
  __shared__ unsigned long long s_red[2];
  const bool route = r.x_perm != nullptr;    // block-uniform
  if (route) {
    for (int i = threadIdx.x; i < WPB * E; i += blockDim.x) s_wcnt[i / E][i % E] = 0;
    if (threadIdx.x < 2) s_red[threadIdx.x] = 0;
  }
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t q = (int64_t)blockIdx.x * WPB + warp;   // this warp's group of rows
  const int64_t t0 = RPW * q;
  const int row = lane / E;              // 0..RPW-1
  const int e_me = lane % E;             // expert held by this lane after the reduce
  const int64_t t = t0 + row;
  const bool row_ok = t < n;
  const int slot = e_me;
  bool valid = false;                    // (t, slot) is an active pair
  int my_e = 0;
  if (t0 < n) {
    int32_t d_last = 0, d_cid = -1;
    uint8_t d_primed = 1, d_red = 0;
    const bool d_lane = d.on && d.strategy != DICE_COND_OFF && row_ok && slot < k;
    if (d_lane) {
      d_last = d.last[t];
      d_primed = d.primed[t];
      d_red = d.reduced[t * k + slot];
      if (d.strict) d_cid = d.cached_ids[t * k + slot];
    }
    const float* rp[RPW];
#pragma unroll
    for (int i = 0; i < RPW; ++i) rp[i] = u + (t0 + i < n ? t0 + i : t0) * hp;
    float2 acc[NP][E];
#pragma unroll
    for (int pp = 0; pp < NP; ++pp)
#pragma unroll
      for (int e = 0; e < E; ++e) acc[pp][e] = make_float2(0.f, 0.f);
    for (int base = 0; base < hp; base += 128 * CH) {
      float4 x[RPW][CH];
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        const int c = base + 128 * j + lane * 4;
#pragma unroll
        for (int i = 0; i < RPW; ++i)
          x[i][j] = c < hp ? ldg_stream_f4(rp[i] + c)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        const int c = base + 128 * j + lane * 4;
        if (c >= hp) break;
        if (route) {
#pragma unroll
          for (int i = 0; i < RPW; ++i) {
            __nv_bfloat162 lo = __floats2bfloat162_rn(x[i][j].x, x[i][j].y);
            __nv_bfloat162 hi = __floats2bfloat162_rn(x[i][j].z, x[i][j].w);
            *reinterpret_cast<uint2*>(s_rows + (int64_t)(warp * RPW + i) * hp + c) =
                make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
          }
        }
        float2 p[NP][4];
#pragma unroll
        for (int pp = 0; pp < NP; ++pp) {
          const float4 a = x[2 * pp][j], b = x[2 * pp + 1][j];
          p[pp][0] = make_float2(a.x, b.x); p[pp][1] = make_float2(a.y, b.y);
          p[pp][2] = make_float2(a.z, b.z); p[pp][3] = make_float2(a.w, b.w);
        }
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const float4 w = __ldg(reinterpret_cast<const float4*>(wt + (int64_t)e * hp + c));
#pragma unroll
          for (int pp = 0; pp < NP; ++pp) acc[pp][e] = __ffma2_rn(p[pp][0], make_float2(w.x, w.x), acc[pp][e]);
#pragma unroll
          for (int pp = 0; pp < NP; ++pp) acc[pp][e] = __ffma2_rn(p[pp][1], make_float2(w.y, w.y), acc[pp][e]);
#pragma unroll
          for (int pp = 0; pp < NP; ++pp) acc[pp][e] = __ffma2_rn(p[pp][2], make_float2(w.z, w.z), acc[pp][e]);
#pragma unroll
          for (int pp = 0; pp < NP; ++pp) acc[pp][e] = __ffma2_rn(p[pp][3], make_float2(w.w, w.w), acc[pp][e]);
        }
      }
    }
    float a[32];                           // index = row * E + e
#pragma unroll
    for (int pp = 0; pp < NP; ++pp)
#pragma unroll
      for (int e = 0; e < E; ++e) {
        a[(2 * pp) * E + e] = acc[pp][e].x;
        a[(2 * pp + 1) * E + e] = acc[pp][e].y;
      }
    tr_level<32>(a, lane, 16); tr_level<16>(a, lane, 8); tr_level<8>(a, lane, 4);
    tr_level<4>(a, lane, 2); tr_level<2>(a, lane, 1);
    const float logit = a[0];              // row (lane / E), expert (lane % E)
    const bool bad = !isfinite(logit) && row_ok;
    if (__any_sync(0xffffffffu, bad) && lane == 0) record_nonfinite(status, step, layer);
    float mx = logit;
#pragma unroll
    for (int off = 1; off < E; off <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    const float ex = expf(logit - mx);
    float sum = ex;
#pragma unroll
    for (int off = 1; off < E; off <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
    const float sc = ex / sum;
    const int rowbase = row * E;
    int rank = 0;
#pragma unroll
    for (int qe = 0; qe < E; ++qe) {
      const float sq = __shfl_sync(0xffffffffu, sc, rowbase + qe);
      rank += (sq > sc) || (sq == sc && qe < e_me);
    }
    if (scores != nullptr && row_ok) scores[t * E + e_me] = sc;
    const unsigned rowmask = (E == 32 ? 0xFFFFFFFFu : ((1u << E) - 1u)) << rowbase;
    float psum = 0.f, my_s = 0.f;
    for (int j = 0; j < k; ++j) {
      const unsigned m = __ballot_sync(0xffffffffu, rank == j) & rowmask;
      const int src = __ffs(m) - 1;
      const float sj = __shfl_sync(0xffffffffu, sc, src);
      psum += sj;
      if (slot == j) { my_s = sj; my_e = src % E; }
    }
    if (slot < k && row_ok) {
      ids[t * k + slot] = my_e;
      gates[t * k + slot] = my_s / psum;
    }
    bool my_act = true;
    if (d.on && slot < k && row_ok) {
      if (d.strategy == DICE_COND_OFF) {
        d.active[t * k + slot] = 1;
        d.write[t * k + slot] = 0;
      } else {
        const bool due = d.force || !d_primed || (step - d_last) >= d.R;
        bool red = d_red != 0;
        if (due) {
          if (d.strategy == DICE_COND_LOW_SCORE) red = slot >= 1;
          else if (d.strategy == DICE_COND_HIGH_SCORE) red = slot == 0;
          else red = slot != (int)(splitmix_at(d.key, (uint64_t)t + 1) % (uint64_t)k);
          d.reduced[t * k + slot] = red;
          if (slot == 0) { d.last[t] = step; d.primed[t] = 1; }
        }
        bool act = !red || due;
        bool wr = red && due;
        if (d.strict && red && !due && my_e != d_cid) { act = true; wr = true; }
        d.active[t * k + slot] = act;
        d.write[t * k + slot] = wr;
        my_act = act;
      }
    }
    valid = slot < k && row_ok && my_act;
  }
  if (!route) return;
  // ---------------------------------------------------------- permute
  const unsigned peers = __match_any_sync(0xffffffffu, valid ? my_e : -1);
  const int rank_in_warp = __popc(peers & ((1u << lane) - 1));
  __syncthreads();                       // s_wcnt zeroed by every warp's view
  if (valid && rank_in_warp == 0) s_wcnt[warp][my_e] = __popc(peers);
  {
    bool remote = false;
    if (valid && r.devices > 1)
      remote = (int)((t * r.devices) / r.rows_total) != my_e / (E / r.devices);
    const unsigned nv = __popc(__ballot_sync(0xffffffffu, valid));
    const unsigned nr = __popc(__ballot_sync(0xffffffffu, remote));
    if (lane == 0 && nv) atomicAdd(&s_red[0], (unsigned long long)nv);
    if (lane == 0 && nr) atomicAdd(&s_red[1], (unsigned long long)nr);
  }
  __syncthreads();
#pragma unroll
  for (int e = warp; e < E; e += WPB) {
    // warp w owns experts w, w + WPB, ...: the block's count of the expert
    // (exclusive prefix over the warps back into s_wcnt) and ONE atomic add
    // on the expert's row counter, whose return value is the block's offset in
    // the region. Blocks take their offsets in arrival order, so the order of
    // rows within an expert region varies between launches; every row's
    // expert-FFN output depends on that row alone, so no value does. (Offsets
    // in block order need the predecessors' counts: a look-back chain measured
    // 14 us slower at 8192 rows, a grid-wide count barrier 5 us slower and
    // only valid while every block is resident.)
    const int c = lane < WPB ? s_wcnt[lane][e] : 0;
    int inc = c;
#pragma unroll
    for (int off = 1; off < WPB; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, off);
      if (lane >= off) inc += y;
    }
    const unsigned acc_e = (unsigned)__shfl_sync(0xffffffffu, inc, WPB - 1);
    if (lane < WPB) s_wcnt[lane][e] = inc - c;
    unsigned base = 0;
    if (lane == 0 && acc_e) base = atomicAdd(&r.state[1 + e], acc_e);
    if (lane == 0) s_base[e] = (int)(e * r.cap) + (int)base;
  }
  __syncthreads();
  if (t0 < n && slot < k && row_ok) {
    const int p = valid ? s_base[my_e] + s_wcnt[warp][my_e] + rank_in_warp : -1;
    r.pos[t * k + slot] = p;
    if (valid) r.row_pair[p] = (int32_t)(t * k + slot);
    s_pos[(warp * RPW + row) * k + slot] = p;
  } else if (slot < k) {
    s_pos[(warp * RPW + row) * k + slot] = -1;
  }
  // the staged rows were written through the generic proxy; the bulk copies
  // below read them through the async proxy
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  // copy the staged bf16 rows to their permuted positions: one bulk async
  // copy (TMA engine, smem -> global) per active pair, issued by one thread
  // per pair; the issuing threads wait until their copies have read smem
  for (int qq = threadIdx.x; qq < TPB * k; qq += blockDim.x) {
    const int p = s_pos[qq];
    if (p < 0) continue;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 ::"l"(r.x_perm + (int64_t)p * hp),
                   "r"((uint32_t)__cvta_generic_to_shared(s_rows + (int64_t)(qq / k) * hp)),
                   "r"(hp * 2)
                 : "memory");
  }
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  if (threadIdx.x == 0) {
    if (s_red[0]) atomicAdd(reinterpret_cast<unsigned long long*>(&r.counters[0]), s_red[0]);
    if (s_red[1]) atomicAdd(reinterpret_cast<unsigned long long*>(&r.counters[1]), s_red[1]);
  }
  // the last block to finish: every row counter is final -> the 256-row tile
  // prefix, the padding rows of every region, and the counters reset for the
  // next launch
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_fin = atomicAdd(&r.state[0], 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_fin) return;
  __threadfence();
  if (threadIdx.x < E) s_tot[threadIdx.x] = (int)ld_relaxed_u32(&r.state[1 + threadIdx.x]);
  __syncthreads();
  if (threadIdx.x == 0) {
    int tiles = 0;
    for (int e = 0; e < E; ++e) {
      r.tile_offsets[e] = tiles;
      tiles += (s_tot[e] + kRowTileR - 1) / kRowTileR;
    }
    r.tile_offsets[E] = tiles;
  }
  for (int e = 0; e < E; ++e) {
    const int64_t b0 = e * r.cap + s_tot[e];
    const int64_t b1 = e * r.cap + (s_tot[e] + kRowTileR - 1) / kRowTileR * kRowTileR;
    for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) r.row_pair[i] = -1;
  }
  if (threadIdx.x <= E) r.state[threadIdx.x] = 0;
}


// ------------------------------------------------------------- permute
// Pairs are visited in token-major order p = t*k + s; within an expert the
// rows are ordered by p, a deterministic order (the GEMM rows are independent,
// so the grouping order of routed_rows, model.py:267-275, does not change any
// value). Block b owns pairs [b*1024, (b+1)*1024): the count kernel writes the
// per-(block, expert) counts; the scatter kernel derives its block prefix and
// the 256-row-padded expert bases from all blocks' counts (no grid-wide sync)
// and assigns positions from warp-level match ranks.
constexpr int kPermBlock = 1024;
constexpr int kRowTile = 256;  // expert groups padded to the CTA-pair GEMM's 256-row tile
// (the EP send plan groups by destination rank with key_div = E/D and row_tile = 1)

__device__ __forceinline__ bool pair_of(int64_t p, int k, const int32_t* ids,
                                        const uint8_t* active, int key_div, int& e, int64_t& t,
                                        int& s) {
  t = p / k;
  s = (int)(p - t * k);
  e = ids[p];
  const bool ok = e >= 0 && (active == nullptr || active[p] != 0);
  if (key_div > 1) e /= key_div;
  return ok;
}

// Rank of this thread's pair among earlier pairs of the same expert in its
// block (wcnt: per-warp counts turned into exclusive prefixes over warps).
__device__ __forceinline__ int block_rank(bool valid, int e, int E, int (*wcnt)[64]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 32 * E; i += blockDim.x) wcnt[i / E][i % E] = 0;
  __syncthreads();
  const int key = valid ? e : -1;
  const unsigned peers = __match_any_sync(0xffffffffu, key);
  const int rank_in_warp = __popc(peers & ((1u << lane) - 1));
  if (valid && rank_in_warp == 0) wcnt[warp][e] = __popc(peers);
  __syncthreads();
  if (threadIdx.x < E) {
    int acc = 0;
    for (int w = 0; w < 32; ++w) { const int c = wcnt[w][threadIdx.x]; wcnt[w][threadIdx.x] = acc; acc += c; }
  }
  __syncthreads();
  return valid ? wcnt[warp][e] + rank_in_warp : 0;
}

__global__ void __launch_bounds__(kPermBlock) permute_count_kernel(
    const int32_t* __restrict__ ids, const uint8_t* __restrict__ active, int64_t n, int k, int E,
    long long* counters, int devices, int64_t row0, int64_t rows_total, int32_t* block_counts,
    int key_div, int experts_total) {
  pdl_enter();
  __shared__ int cnt[64];
  __shared__ unsigned long long red[2];
  if (threadIdx.x < 64) cnt[threadIdx.x] = 0;
  if (threadIdx.x < 2) red[threadIdx.x] = 0;
  __syncthreads();
  const int64_t P = n * k;
  const int64_t p = (int64_t)blockIdx.x * kPermBlock + threadIdx.x;
  int e = 0, s = 0;
  int64_t t = 0;
  bool valid = false;
  int e_raw = -1;
  if (p < P) { valid = pair_of(p, k, ids, active, key_div, e, t, s); e_raw = ids[p]; }
  const unsigned peers = __match_any_sync(0xffffffffu, valid ? e : -1);
  const int lane = threadIdx.x & 31;
  if (valid && __popc(peers & ((1u << lane) - 1)) == 0) atomicAdd(&cnt[e], __popc(peers));
  // byte plan: active pairs whose expert device differs from the token home (cluster.py:75-90)
  bool remote = false;
  if (valid && devices > 1) {
    const int home = (int)(((row0 + t) * devices) / rows_total);
    const int edev = e_raw / (experts_total / devices);
    remote = home != edev;
  }
  const unsigned nv = __popc(__ballot_sync(0xffffffffu, valid));
  const unsigned nr = __popc(__ballot_sync(0xffffffffu, remote));
  if (lane == 0 && nv) atomicAdd(&red[0], (unsigned long long)nv);
  if (lane == 0 && nr) atomicAdd(&red[1], (unsigned long long)nr);
  __syncthreads();
  if (threadIdx.x < E) block_counts[(int64_t)blockIdx.x * E + threadIdx.x] = cnt[threadIdx.x];
  if (threadIdx.x == 0 && counters != nullptr) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&counters[0]), red[0]);
    atomicAdd(reinterpret_cast<unsigned long long*>(&counters[1]), red[1]);
  }
}

__global__ void __launch_bounds__(kPermBlock) permute_scatter_kernel(
    const int32_t* __restrict__ ids, const uint8_t* __restrict__ active, int64_t n, int k, int E,
    int32_t* pos, const int32_t* __restrict__ block_counts, int32_t* tile_offsets, int key_div,
    int row_tile, int32_t* row_pair, int count_rows, int rows_per_block) {
  pdl_enter();
  __shared__ int wcnt[32][64];
  __shared__ int base[64];
  // count rows: one per block of the counting pass (the count kernel: one per
  // scatter block; the gate's fused counting: one per 32 tokens)
  const int first_mine = (int)blockIdx.x * rows_per_block;
  if (E == 8 && blockDim.x == 1024) {
    // 128 row-strided partial sums per expert (thread = 8 part + e), reduced
    // over the 4 parts of a warp by shuffles, then over the 32 warps in smem:
    // no thread walks the count rows serially (the gate's fused counting
    // produces one row per 32 tokens: 256 rows at 8192 tokens)
    __shared__ int red_b[32][8], red_t[32][8];
    const int e = threadIdx.x & 7, part = threadIdx.x >> 3;
    int before = 0, total = 0;
    for (int b = part; b < count_rows; b += 128) {
      const int c = block_counts[(int64_t)b * 8 + e];
      if (b < first_mine) before += c;
      total += c;
    }
#pragma unroll
    for (int off = 8; off < 32; off <<= 1) {
      before += __shfl_xor_sync(0xffffffffu, before, off);
      total += __shfl_xor_sync(0xffffffffu, total, off);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane < 8) { red_b[warp][lane] = before; red_t[warp][lane] = total; }
    __syncthreads();
    if (threadIdx.x < 8) {
      int b = 0, t = 0;
      for (int w = 0; w < 32; ++w) { b += red_b[w][threadIdx.x]; t += red_t[w][threadIdx.x]; }
      wcnt[0][threadIdx.x] = t;
      base[threadIdx.x] = b;
    }
  } else if (threadIdx.x < E) {
    int before = 0, total = 0;
    for (int b = 0; b < count_rows; ++b) {
      const int c = block_counts[(int64_t)b * E + threadIdx.x];
      if (b < first_mine) before += c;
      total += c;
    }
    wcnt[0][threadIdx.x] = total;
    base[threadIdx.x] = before;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int tiles = 0;
    for (int ex = 0; ex < E; ++ex) {
      if (blockIdx.x == 0) tile_offsets[ex] = tiles;
      base[ex] += tiles * row_tile;
      tiles += (wcnt[0][ex] + row_tile - 1) / row_tile;
    }
    if (blockIdx.x == 0) tile_offsets[E] = tiles;
  }
  __syncthreads();
  if (row_pair != nullptr && blockIdx.x == 0) {
    // padding rows of every expert group map to no pair (block 0's bases are
    // the group starts)
    for (int ex = 0; ex < E; ++ex) {
      const int cnt = wcnt[0][ex];
      const int pad_end = base[ex] + (cnt + row_tile - 1) / row_tile * row_tile;
      for (int r = base[ex] + cnt + threadIdx.x; r < pad_end; r += blockDim.x) row_pair[r] = -1;
    }
  }
  __syncthreads();   // block_rank() reuses wcnt[0][*] (the group totals read above)
  const int64_t P = n * k;
  const int64_t p = (int64_t)blockIdx.x * kPermBlock + threadIdx.x;
  int e = 0, s = 0;
  int64_t t = 0;
  bool valid = false;
  const bool in_range = p < P;
  if (in_range) valid = pair_of(p, k, ids, active, key_div, e, t, s);
  const int r = block_rank(valid, e, E, wcnt);
  if (in_range) pos[p] = valid ? base[e] + r : -1;
  if (row_pair != nullptr && valid) row_pair[base[e] + r] = (int32_t)p;   // row -> pair
}

// Row gather x_perm[pos[t, s]] = u16[t]: one warp per (token, slot) pair,
// 16-byte vector copies, grid over all pairs.
__global__ void __launch_bounds__(256) permute_gather_kernel(
    const int32_t* __restrict__ pos, int64_t pairs, const uint16_t* __restrict__ u16, int k,
    int hp, uint16_t* __restrict__ x_perm) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const int vec = hp / 8;
  for (int64_t q = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; q < pairs;
       q += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int d = pos[q];
    if (d < 0) continue;
    const int64_t t = q / k;
    const uint4* src = reinterpret_cast<const uint4*>(u16 + t * hp);
    uint4* out = reinterpret_cast<uint4*>(x_perm + (int64_t)d * hp);
    uint4 v[5];
#pragma unroll
    for (int j = 0; j < 5; ++j) if (lane + 32 * j < vec) v[j] = src[lane + 32 * j];
#pragma unroll
    for (int j = 0; j < 5; ++j) if (lane + 32 * j < vec) out[lane + 32 * j] = v[j];
    for (int c = lane + 160; c < vec; c += 32) out[c] = src[c];
  }
}

// ------------------------------------------------------- cache assemble
// One thread per (token, 8 columns). Slots are visited left to right and
// accumulated in fp32 (model.py:295-297). Active pairs read the fresh expert
// row; inactive pairs read the cached row and gate (policies.py:197-202);
// write pairs persist row / gate / id (policies.py:203-207). write implies
// active, so no thread reads a cache entry another thread writes.
template <int KMAX>
__global__ void __launch_bounds__(256) cache_assemble_kernel(
    const uint16_t* __restrict__ y, const int32_t* __restrict__ pos,
    const uint8_t* __restrict__ active, const uint8_t* __restrict__ write,
    const float* __restrict__ gates, const int32_t* __restrict__ ids, int64_t n, int k, int hp,
    uint16_t* cache_rows, float* cache_gates, int32_t* cache_ids, float* routed, float* rows_out,
    float* gates_out) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const int vec = hp / 8;
  for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < n;
       t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    // per-slot metadata, loaded once per warp
    const uint16_t* src[KMAX];
    float g[KMAX];
    bool wr[KMAX];
    for (int s = 0; s < k && s < KMAX; ++s) {
      const int64_t ps = t * k + s;
      const bool act = active == nullptr || active[ps] != 0;
      wr[s] = act && write != nullptr && write[ps] != 0;
      if (act) {
        src[s] = y + (int64_t)pos[ps] * hp;
        g[s] = gates[ps];
      } else if (cache_rows != nullptr) {
        src[s] = cache_rows + ((int64_t)s * n + t) * hp;
        g[s] = cache_gates[ps];
      } else {  // no cache: inactive pairs stay zero (routed_rows, model.py:262)
        src[s] = nullptr;
        g[s] = 0.f;
      }
      if (lane == 0) {
        if (wr[s]) { cache_gates[ps] = g[s]; cache_ids[ps] = ids[ps]; }
        if (gates_out != nullptr) gates_out[ps] = g[s];
      }
    }
    constexpr int CH = 3;  // 8-column chunks per lane per batch (k*CH loads in flight)
    for (int base = 0; base < vec; base += 32 * CH) {
      uint4 raw[KMAX][CH];
      for (int s = 0; s < k && s < KMAX; ++s) {
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          const int c8 = base + 32 * j + lane;
          raw[s][j] = (src[s] != nullptr && c8 < vec)
                          ? *reinterpret_cast<const uint4*>(src[s] + c8 * 8)
                          : make_uint4(0, 0, 0, 0);
        }
      }
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        const int c8 = base + 32 * j + lane;
        if (c8 >= vec) break;
        const int c = c8 * 8;
        float acc[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = 0.f;
        for (int s = 0; s < k && s < KMAX; ++s) {
          if (wr[s]) *reinterpret_cast<uint4*>(cache_rows + ((int64_t)s * n + t) * hp + c) = raw[s][j];
          const uint16_t* hv = reinterpret_cast<const uint16_t*>(&raw[s][j]);
          float v[8];
#pragma unroll
          // acc + round(g * row): the same two roundings an order-free
          // (atomic) accumulation of the k <= 2 slot terms produces
          for (int q = 0; q < 8; ++q) {
            v[q] = bf16_bits_to_f32(hv[q]);
            acc[q] = __fadd_rn(acc[q], __fmul_rn(g[s], v[q]));
          }
          if (rows_out != nullptr) {
            float4* ro = reinterpret_cast<float4*>(rows_out + ((int64_t)s * n + t) * hp + c);
            ro[0] = make_float4(v[0], v[1], v[2], v[3]);
            ro[1] = make_float4(v[4], v[5], v[6], v[7]);
          }
        }
        float4* o = reinterpret_cast<float4*>(routed + t * hp + c);
        o[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
        o[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
      }
    }
  }
}

// ---------------------------------------------------------------- combine
__global__ void combine_kernel(const float* __restrict__ base, const float* __restrict__ rows,
                               const float* __restrict__ gates, const float* __restrict__ residual,
                               int64_t n, int k, int hp, float* out, __nv_bfloat16* out16) {
  pdl_enter();
  const int vec = hp / 4;
  const int64_t total = n * vec;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / vec;
    const int c = (int)(i - t * vec) * 4;
    float4 a = *reinterpret_cast<const float4*>(base + t * hp + c);
    for (int s = 0; s < k; ++s) {
      const float g = gates[t * k + s];
      const float4 r = *reinterpret_cast<const float4*>(rows + ((int64_t)s * n + t) * hp + c);
      a.x += g * r.x; a.y += g * r.y; a.z += g * r.z; a.w += g * r.w;
    }
    if (residual != nullptr) {
      const float4 u = *reinterpret_cast<const float4*>(residual + t * hp + c);
      a = make_float4(u.x + a.x, u.y + a.y, u.z + a.z, u.w + a.w);
    }
    *reinterpret_cast<float4*>(out + t * hp + c) = a;
    if (out16 != nullptr) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(a.x, a.y), hi = __floats2bfloat162_rn(a.z, a.w);
      uint2 w = make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
      *reinterpret_cast<uint2*>(out16 + t * hp + c) = w;
    }
  }
}

// Consume without shared experts (S = 0): h = u + ((0 + g_0 row_0) + g_1 row_1 ...)
// over the layer's bf16 pair rows [k, n, hp] and gates [n, k] (schedules.py:308-317,
// model.py:279-298), in the shared-GEMM consume epilogue's arithmetic order.
__global__ void consume_rows_kernel(const float* __restrict__ residual,
                                    const uint16_t* __restrict__ rows,
                                    const float* __restrict__ gates, int64_t n, int k, int hp,
                                    float* out, __nv_bfloat16* out16) {
  pdl_enter();
  const int vec = hp / 4;
  const int64_t total = n * vec;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / vec;
    const int c = (int)(i - t * vec) * 4;
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < k; ++s) {
      const float g = gates[t * k + s];
      const uint2 w = *reinterpret_cast<const uint2*>(rows + ((int64_t)s * n + t) * hp + c);
      const float r0 = bf16_bits_to_f32(w.x & 0xFFFFu), r1 = bf16_bits_to_f32(w.x >> 16);
      const float r2 = bf16_bits_to_f32(w.y & 0xFFFFu), r3 = bf16_bits_to_f32(w.y >> 16);
      a = make_float4(__fadd_rn(a.x, __fmul_rn(g, r0)), __fadd_rn(a.y, __fmul_rn(g, r1)),
                      __fadd_rn(a.z, __fmul_rn(g, r2)), __fadd_rn(a.w, __fmul_rn(g, r3)));
    }
    const float4 u = *reinterpret_cast<const float4*>(residual + t * hp + c);
    a = make_float4(__fadd_rn(u.x, a.x), __fadd_rn(u.y, a.y), __fadd_rn(u.z, a.z),
                    __fadd_rn(u.w, a.w));
    *reinterpret_cast<float4*>(out + t * hp + c) = a;
    if (out16 != nullptr) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(a.x, a.y), hi = __floats2bfloat162_rn(a.z, a.w);
      *reinterpret_cast<uint2*>(out16 + t * hp + c) =
          make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
    }
  }
}

// ---------------------------------------------------------------- denoise
__global__ void denoise_kernel(float* x, __nv_bfloat16* x16, const float* __restrict__ y, float eta,
                               int64_t count4, int32_t* status, int step) {
  pdl_enter();
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count4;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 a = reinterpret_cast<float4*>(x)[i];
    const float4 b = reinterpret_cast<const float4*>(y)[i];
    a.x = a.x - eta * b.x; a.y = a.y - eta * b.y; a.z = a.z - eta * b.z; a.w = a.w - eta * b.w;
    bad |= !(isfinite(a.x) && isfinite(a.y) && isfinite(a.z) && isfinite(a.w));
    reinterpret_cast<float4*>(x)[i] = a;
    if (x16 != nullptr) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(a.x, a.y), hi = __floats2bfloat162_rn(a.z, a.w);
      reinterpret_cast<uint2*>(x16)[i] =
          make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) record_nonfinite(status, step, -1);
}

__global__ void pack_rows_kernel(const float* __restrict__ in, int64_t n, int cols, int64_t ld_in,
                                 int hp, float* out32, __nv_bfloat16* out16) {
  pdl_enter();
  const int64_t total = n * hp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / hp;
    const int c = (int)(i - t * hp);
    const float v = c < cols ? in[t * ld_in + c] : 0.f;
    if (out32 != nullptr) out32[i] = v;
    if (out16 != nullptr) out16[i] = __float2bfloat16_rn(v);
  }
}


// ------------------------------------------------------- step similarity
// Adjacent-step drift of one layer's MoE input and its routing
// (step_similarity / _cosine, model.py:308-346): fp64 sums dot(a, b), |a|^2,
// |b|^2 over the first `cols` columns of n rows, and the number of rows whose
// top-1 expert agrees (top_a[t * top_stride] vs ids_b[t * k]). Deterministic:
// a fixed grid of kSimBlocks blocks, each thread owning a fixed set of
// elements, fixed-order tree reductions, then one block summing the block
// partials in block order. roll != 0 also stores b into a and b's top-1 into
// top_a (the runner's previous-step buffers), after reading them.
constexpr int kSimBlocks = 296;
constexpr int kSimThreads = 256;

__device__ __forceinline__ void sim_block_sum(double (&v)[4], double* s_red /*[4][8]*/) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v[j] += __shfl_down_sync(0xffffffffu, v[j], off);
    if (lane == 0) s_red[j * 8 + warp] = v[j];
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    double acc = 0.0;
    for (int w = 0; w < kSimThreads / 32; ++w) acc += s_red[threadIdx.x * 8 + w];
    v[threadIdx.x] = acc;    // thread j holds sum j
  }
}

__global__ void __launch_bounds__(kSimThreads) similarity_partial_kernel(
    float* a, const float* b, int64_t n, int cols, int64_t lda, int64_t ldb, int32_t* top_a,
    int64_t top_stride, const int32_t* __restrict__ ids_b, int k, int roll, double* part) {
  __shared__ double s_red[4 * 8];
  pdl_enter();
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  const bool vec = (cols % 4 == 0) && (lda % 4 == 0) && (ldb % 4 == 0);
  for (int64_t t = blockIdx.x; t < n; t += gridDim.x) {
    float* ar = a + t * lda;
    const float* br = b + t * ldb;
    if (vec) {
      for (int c = threadIdx.x * 4; c < cols; c += kSimThreads * 4) {
        const float4 x = *reinterpret_cast<const float4*>(ar + c);
        const float4 y = *reinterpret_cast<const float4*>(br + c);
        v[0] = fma((double)x.x, (double)y.x, v[0]); v[1] = fma((double)x.x, (double)x.x, v[1]);
        v[2] = fma((double)y.x, (double)y.x, v[2]);
        v[0] = fma((double)x.y, (double)y.y, v[0]); v[1] = fma((double)x.y, (double)x.y, v[1]);
        v[2] = fma((double)y.y, (double)y.y, v[2]);
        v[0] = fma((double)x.z, (double)y.z, v[0]); v[1] = fma((double)x.z, (double)x.z, v[1]);
        v[2] = fma((double)y.z, (double)y.z, v[2]);
        v[0] = fma((double)x.w, (double)y.w, v[0]); v[1] = fma((double)x.w, (double)x.w, v[1]);
        v[2] = fma((double)y.w, (double)y.w, v[2]);
        if (roll) *reinterpret_cast<float4*>(ar + c) = y;
      }
    } else {
      for (int c = threadIdx.x; c < cols; c += kSimThreads) {
        const double x = ar[c], y = br[c];
        v[0] = fma(x, y, v[0]); v[1] = fma(x, x, v[1]); v[2] = fma(y, y, v[2]);
        if (roll) ar[c] = br[c];
      }
    }
    if (threadIdx.x == 0) {
      const int32_t tb = ids_b[t * k];
      v[3] += top_a[t * top_stride] == tb ? 1.0 : 0.0;
      if (roll) top_a[t * top_stride] = tb;
    }
  }
  sim_block_sum(v, s_red);
  if (threadIdx.x < 4) part[(int64_t)threadIdx.x * gridDim.x + blockIdx.x] = v[threadIdx.x];
}

__global__ void __launch_bounds__(kSimThreads) similarity_final_kernel(const double* part,
                                                                       int parts, double* out) {
  __shared__ double s_red[4 * 8];
  pdl_enter();
  double v[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    double acc = 0.0;
    for (int i = threadIdx.x; i < parts; i += kSimThreads) acc += part[(int64_t)j * parts + i];
    v[j] = acc;
  }
  sim_block_sum(v, s_red);
  if (threadIdx.x < 4) out[threadIdx.x] = v[threadIdx.x];
}

static int grid_for(int64_t work, int threads) {
  int64_t g = (work + threads - 1) / threads;
  const int64_t cap = 148 * 16;
  if (g > cap) g = cap;
  return g < 1 ? 1 : (int)g;
}

static inline int launch_ok() { return cudaGetLastError() == cudaSuccess ? DICE_OK : DICE_ERR_CUDA; }

int permute_launch(const int32_t* ids, const uint8_t* active, int64_t n, int k, int groups,
                   int key_div, int row_tile, int experts_total, const uint16_t* rows, int hp,
                   uint16_t* x_perm, int32_t* pos, int32_t* tile_offsets, int64_t* counters,
                   int devices, int64_t row0, int64_t rows_total, int32_t* scratch,
                   cudaStream_t s, int32_t* row_pair) {
  const int64_t P = n * k;
  const int blocks = (int)((P + kPermBlock - 1) / kPermBlock);
  if (blocks == 0) {
    cudaMemsetAsync(tile_offsets, 0, sizeof(int32_t) * (groups + 1), s);
    return launch_ok();
  }
  launch_pdl(permute_count_kernel, dim3(blocks), dim3(kPermBlock), 0, s, ids, active, n, k, groups,
                                                     reinterpret_cast<long long*>(counters), devices,
                                                     row0, rows_total, scratch, key_div,
                                                     experts_total);
  launch_pdl(permute_scatter_kernel, dim3(blocks), dim3(kPermBlock), 0, s, ids, active, n, k, groups, pos, scratch,
                                                       tile_offsets, key_div, row_tile, row_pair, blocks, 1);
  if (x_perm != nullptr)
    launch_pdl(permute_gather_kernel, dim3(grid_for(P * 32, 256)), dim3(256), 0, s, pos, P, rows, k, hp, x_perm);
  return launch_ok();
}

}  // namespace dice

using namespace dice;

extern "C" {

int dice_version(void) { return 100; }

int dice_event_create(void** event) {
  cudaEvent_t e;
  if (cudaEventCreate(&e) != cudaSuccess) return DICE_ERR_CUDA;
  *event = (void*)e;
  return DICE_OK;
}

int dice_event_destroy(void* event) {
  return cudaEventDestroy((cudaEvent_t)event) == cudaSuccess ? DICE_OK : DICE_ERR_CUDA;
}

// Records as an event node when the stream is being captured into a CUDA
// graph (cudaEventRecordExternal), so graph replays keep per-kernel timing.
int dice_event_record(void* event, void* stream) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing((cudaStream_t)stream, &st);
  const unsigned flags = st == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : 0;
  return cudaEventRecordWithFlags((cudaEvent_t)event, (cudaStream_t)stream, flags) == cudaSuccess
             ? DICE_OK : DICE_ERR_CUDA;
}

int dice_event_elapsed_ms(void* start, void* end, float* ms) {
  return cudaEventElapsedTime(ms, (cudaEvent_t)start, (cudaEvent_t)end) == cudaSuccess
             ? DICE_OK : DICE_ERR_CUDA;
}

int dice_status_reset(int32_t* status, void* stream) {
  status_reset_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(status);
  return launch_ok();
}

int dice_splitmix_fill(uint64_t seed, uint64_t start, int64_t rows, int64_t cols, double halfwidth,
                       int transpose, int out_dtype, void* out, int64_t ld, void* stream) {
  if (rows < 0 || cols < 0 || out_dtype < 0 || out_dtype > 2) return DICE_ERR_CONTRACT;
  if (rows * cols == 0) return DICE_OK;
  splitmix_fill_kernel<<<grid_for(rows * cols, 256), 256, 0, (cudaStream_t)stream>>>(
      seed, start, rows, cols, halfwidth, transpose, out_dtype, out, ld);
  return launch_ok();
}

int dice_splitmix_bits(uint64_t seed, uint64_t start, int64_t count, uint64_t* out, void* stream) {
  if (count < 0) return DICE_ERR_CONFIG;
  if (count == 0) return DICE_OK;
  splitmix_bits_kernel<<<grid_for(count, 256), 256, 0, (cudaStream_t)stream>>>(seed, start, count, out);
  return launch_ok();
}

namespace {
int gate_topk_launch(const float* u, const float* w_gate_t, int64_t n, int hp, int E, int k,
                     int32_t* ids, float* gates, float* scores, int32_t* status, int step,
                     int layer, const DecideArgs& d, cudaStream_t s,
                     const RouteArgs& ra = RouteArgs{}) {
  if (E < 1 || E > 64 || k < 1 || k > E || hp % 64 != 0) return DICE_ERR_CONTRACT;
  if (n == 0) return DICE_OK;
  // the fused permute lives in the E = 8 / 16 router kernel only
  if (ra.x_perm != nullptr && ((E != 8 && E != 16) || k > E)) return DICE_ERR_CONTRACT;
  const size_t smem = (size_t)E * hp * sizeof(float);
  const int threads = 512;
  int64_t want = ((n + 1) / 2 + 15) / 16;
  if (smem > 200 * 1024) return DICE_ERR_CONTRACT;
  if ((E == 8 || E == 16) && k <= E) {
    // kRouterWarps warps per block: four rows per warp at E = 8, two at E = 16
    constexpr int WPB = kRouterWarps;
    const int rpw = 32 / E;
    const int64_t gw = ((n + rpw - 1) / rpw + WPB - 1) / WPB;
    const int grid = (int)(gw < 1 ? 1 : gw);
    const size_t rsmem = ra.x_perm != nullptr ? (size_t)WPB * rpw * hp * sizeof(uint16_t) : 0;
    auto kern = E == 8 ? gate4_topk_kernel<8, 3, WPB> : gate4_topk_kernel<16, 3, WPB>;
    if (rsmem > 0) {
      static size_t attr[2] = {0, 0};
      size_t& a = attr[E == 8 ? 0 : 1];
      if (rsmem > a) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsmem) !=
            cudaSuccess)
          return DICE_ERR_CUDA;
        a = rsmem;
      }
    }
    launch_pdl(kern, dim3(grid), dim3(32 * WPB), rsmem, s, u, w_gate_t, n, hp, k, ids, gates,
               scores, status, step, layer, d, ra);
    return launch_ok();
  }
  const int grid = (int)(want < 2 * 148 ? (want < 1 ? 1 : want) : 2 * 148);
#define DICE_GATE(EM)                                                                          \
  {                                                                                            \
    static bool attr = false;                                                                  \
    if (!attr) {                                                                               \
      cudaFuncSetAttribute(gate_topk_kernel<EM>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           200 * 1024);                                                        \
      attr = true;                                                                             \
    }                                                                                          \
    launch_pdl(gate_topk_kernel<EM>, dim3(grid), dim3(threads), smem, s, u, w_gate_t, n, hp, E, k, ids, gates,     \
                                                     scores, status, step, layer);             \
  }
  if (E <= 8) DICE_GATE(8)
  else if (E <= 16) DICE_GATE(16)
  else DICE_GATE(64)
#undef DICE_GATE
  if (d.on) {
    launch_pdl(cond_decide_kernel, dim3(grid_for(n, 256)), dim3(256), 0, s, ids, n, k, d);
  }
  return launch_ok();
}
}  // namespace

int dice_gate_topk(const float* u, const float* w_gate_t, int64_t n, int hp, int E, int k,
                   int32_t* ids, float* gates, float* scores, int32_t* status, int step, int layer,
                   void* stream) {
  const DecideArgs d{0, 0, 0, 1, 0, 0, 0, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  return gate_topk_launch(u, w_gate_t, n, hp, E, k, ids, gates, scores, status, step, layer, d,
                          (cudaStream_t)stream);
}

int dice_gate_topk_decide(const float* u, const float* w_gate_t, int64_t n, int hp, int E, int k,
                          int32_t* ids, float* gates, float* scores, int32_t* status, int step,
                          int layer, int force, int refresh_interval, int strategy, int strict,
                          uint64_t random_key, int32_t* last_refresh, uint8_t* primed,
                          uint8_t* reduced, const int32_t* cached_ids, uint8_t* active,
                          uint8_t* write, void* stream) {
  if (refresh_interval < 1 || strategy < 0 || strategy > 3) return DICE_ERR_CONFIG;
  const DecideArgs d{1, step, force, refresh_interval, strategy, strict, random_key,
                     last_refresh, primed, reduced, cached_ids, active, write};
  return gate_topk_launch(u, w_gate_t, n, hp, E, k, ids, gates, scores, status, step, layer, d,
                          (cudaStream_t)stream);
}

int64_t dice_gate_route_state_words(int64_t n) {
  // finished-block ticket + up to 16 per-expert row counters (uint32), zero
  // between launches (the last block resets them)
  (void)n;
  return 9;
}

int dice_gate_route(const float* u, const float* w_gate_t, int64_t n, int hp, int E, int k,
                    int32_t* ids, float* gates, float* scores, int32_t* status, int step,
                    int layer, int decide, int force, int refresh_interval, int strategy,
                    int strict, uint64_t random_key, int32_t* last_refresh, uint8_t* primed,
                    uint8_t* reduced, const int32_t* cached_ids, uint8_t* active,
                    uint8_t* write, uint16_t* x_perm, int64_t cap, int32_t* pos,
                    int32_t* row_pair, int32_t* tile_offsets, int64_t* counters, int devices,
                    int64_t rows_total, uint64_t* route_state, void* stream) {
  if (decide && (refresh_interval < 1 || strategy < 0 || strategy > 3)) return DICE_ERR_CONFIG;
  if ((E != 8 && E != 16) || k < 1 || k > E || x_perm == nullptr || pos == nullptr || row_pair == nullptr ||
      tile_offsets == nullptr || counters == nullptr || route_state == nullptr || cap < n ||
      cap % kRowTileR != 0 || devices < 1 || E % devices != 0 || rows_total < 1 ||
      (int64_t)(256 / E) * hp * 2 > 200 * 1024 || cap * E > INT32_MAX)
    return DICE_ERR_CONTRACT;
  if (n == 0) {
    cudaMemsetAsync(tile_offsets, 0, sizeof(int32_t) * (E + 1), (cudaStream_t)stream);
    return launch_ok();
  }
  const DecideArgs d{decide ? 1 : 0, step, force, refresh_interval, strategy, strict, random_key,
                     last_refresh, primed, reduced, cached_ids, active, write};
  RouteArgs ra{};
  ra.x_perm = x_perm;
  ra.cap = cap;
  ra.pos = pos;
  ra.row_pair = row_pair;
  ra.tile_offsets = tile_offsets;
  ra.counters = reinterpret_cast<long long*>(counters);
  ra.devices = devices;
  ra.rows_total = rows_total;
  ra.state = reinterpret_cast<unsigned*>(route_state);
  return gate_topk_launch(u, w_gate_t, n, hp, E, k, ids, gates, scores, status, step, layer, d,
                          (cudaStream_t)stream, ra);
}

int dice_cond_decide(const int32_t* ids, int64_t n, int k, int step, int force, int refresh_interval,
                     int strategy, int strict, uint64_t random_key, int32_t* last_refresh,
                     uint8_t* primed, uint8_t* reduced, const int32_t* cached_ids, uint8_t* active,
                     uint8_t* write, void* stream) {
  if (k < 1 || refresh_interval < 1 || strategy < 0 || strategy > 3) return DICE_ERR_CONFIG;
  if (n == 0) return DICE_OK;
  const DecideArgs d{1, step, force, refresh_interval, strategy, strict, random_key, last_refresh,
                     primed, reduced, cached_ids, active, write};
  launch_pdl(cond_decide_kernel, dim3(grid_for(n, 256)), dim3(256), 0, (cudaStream_t)stream, ids, n, k, d);
  return launch_ok();
}

int64_t dice_permute_max_rows(int64_t n, int k, int E) {
  const int64_t tiles = (n * k + (kRowTile - 1) * (int64_t)E + kRowTile - 1) / kRowTile;
  return (tiles < 1 ? 1 : tiles) * kRowTile;
}

int64_t dice_permute_scratch_ints(int64_t n, int k, int E) {
  // per-1024-pair block counts of the counting pass
  const int64_t blocks = (n * k + kPermBlock - 1) / kPermBlock;
  return (blocks < 1 ? 1 : blocks) * E;
}

int dice_route_permute(const int32_t* ids, const uint8_t* active, int64_t n, int k, int E,
                       const uint16_t* u16, int hp, uint16_t* x_perm, int64_t max_rows, int32_t* pos,
                       int32_t* tile_offsets, int64_t* counters, int devices, int64_t row0,
                       int64_t rows_total, int32_t* scratch, int32_t* row_pair, void* stream) {
  if (E < 1 || E > 64 || k < 1 || hp % 64 != 0 || devices < 1 || E % devices != 0)
    return DICE_ERR_CONTRACT;
  if (max_rows < dice_permute_max_rows(n, k, E)) return DICE_ERR_CONTRACT;
  return dice::permute_launch(ids, active, n, k, E, 1, kRowTile, E, u16, hp, x_perm, pos,
                              tile_offsets, counters, devices, row0, rows_total, scratch,
                              (cudaStream_t)stream, row_pair);
}

int dice_expert_gemm1_with_dense(const uint16_t* x_perm, int64_t max_rows, int64_t group_stride,
                                 const uint16_t* w1_t, int E, int hp, int ep,
                                 const int32_t* tile_offsets, uint16_t* hbuf, const uint16_t* A2,
                                 int64_t M2, const uint16_t* B2, int N2, uint16_t* out2,
                                 void* stream) {
  if (E < 1 || E > kMaxGroups || hp % 64 != 0 || ep % 64 != 0 || max_rows % kRowTile != 0 ||
      M2 < 0 || M2 > INT_MAX || N2 % 64 != 0 || group_stride < 0 || group_stride % kRowTile != 0)
    return DICE_ERR_CONTRACT;
  GemmProblem p{};
  // group_stride > 0: expert e's rows at e * group_stride of x_perm (E * group_stride
  // rows); the GELU output hbuf stays tile-compact (max_rows rows)
  p.A = x_perm; p.A_rows = group_stride > 0 ? E * group_stride : max_rows; p.B = w1_t;
  p.M = (int)max_rows; p.N = ep; p.K = hp;
  p.num_groups = E; p.group_tile_offsets = tile_offsets; p.max_m_tiles = (int)(max_rows / kRowTile);
  p.epi_kind = EPI_GELU_BF16;
  p.epi.a_group_stride = group_stride;
  p.epi.out_bf16 = reinterpret_cast<__nv_bfloat16*>(hbuf); p.epi.ld_bf16 = ep;
  GemmProblem q{};
  q.A = A2; q.A_rows = M2; q.B = B2; q.M = (int)M2; q.N = N2; q.K = hp;
  q.num_groups = 1; q.group_tile_offsets = nullptr; q.max_m_tiles = 0;
  q.epi_kind = EPI_GELU_BF16;
  q.epi.out_bf16 = reinterpret_cast<__nv_bfloat16*>(out2); q.epi.ld_bf16 = N2;
  if (M2 == 0) return gemm_bf16(p, (cudaStream_t)stream);
  return gemm_bf16_dual(p, q, (cudaStream_t)stream);
}

int dice_expert_gemm2(const uint16_t* hbuf, int64_t max_rows, const uint16_t* w2_t, int E, int hp,
                      int ep, const int32_t* tile_offsets, uint16_t* y, void* stream) {
  if (E < 1 || E > kMaxGroups || hp % 64 != 0 || ep % 64 != 0 || max_rows % kRowTile != 0)
    return DICE_ERR_CONTRACT;
  GemmProblem q{};
  q.A = hbuf; q.A_rows = max_rows; q.B = w2_t; q.M = (int)max_rows; q.N = hp; q.K = ep;
  q.num_groups = E; q.group_tile_offsets = tile_offsets; q.max_m_tiles = (int)(max_rows / kRowTile);
  q.epi_kind = EPI_STORE_BF16;
  q.epi.out_bf16 = reinterpret_cast<__nv_bfloat16*>(y); q.epi.ld_bf16 = hp;
  return gemm_bf16(q, (cudaStream_t)stream);
}

int dice_expert_gemm2_pairs(const uint16_t* hbuf, int64_t max_rows, const uint16_t* w2_t, int E,
                            int hp, int ep, const int32_t* tile_offsets, const int32_t* row_pair,
                            int64_t pair_group_stride, const float* gates, const int32_t* ids,
                            int k, int64_t n, uint16_t* pair_rows, float* cache_gates,
                            int32_t* cache_ids, void* stream) {
  if (E < 1 || E > kMaxGroups || hp % 64 != 0 || ep % 64 != 0 || max_rows % kRowTile != 0 ||
      k < 1 || n < 0 || row_pair == nullptr || pair_rows == nullptr || pair_group_stride < 0 ||
      (cache_gates != nullptr && gates == nullptr) || (cache_ids != nullptr && ids == nullptr))
    return DICE_ERR_CONTRACT;
  GemmProblem q{};
  q.A = hbuf; q.A_rows = max_rows; q.B = w2_t; q.M = (int)max_rows; q.N = hp; q.K = ep;
  q.num_groups = E; q.group_tile_offsets = tile_offsets; q.max_m_tiles = (int)(max_rows / kRowTile);
  q.epi_kind = EPI_STORE_PAIR;
  q.epi.out_bf16 = reinterpret_cast<__nv_bfloat16*>(pair_rows); q.epi.ld_bf16 = hp;
  q.epi.row_pair = row_pair;
  q.epi.pair_group_stride = pair_group_stride;
  q.epi.pair_gates = gates;
  q.epi.pair_ids = ids;
  q.epi.cache_gates = cache_gates;
  q.epi.cache_ids = cache_ids;
  q.epi.top_k = k;
  q.epi.n_tokens = n;
  return gemm_bf16(q, (cudaStream_t)stream);
}

int dice_gemm_consume(const uint16_t* A, int64_t M, const uint16_t* B, int N, int K,
                      const float* residual, int64_t ld_res, const uint16_t* pair_rows,
                      const float* pair_gates, int k, float* out_f32, int64_t ld_f32,
                      uint16_t* out_bf16, int64_t ld_bf16, void* stream) {
  if (M < 0 || M > INT_MAX || residual == nullptr || k < 0 ||
      (k > 0 && (pair_rows == nullptr || pair_gates == nullptr)))
    return DICE_ERR_CONTRACT;
  if (M == 0) return DICE_OK;
  GemmProblem p{};
  p.A = A; p.A_rows = M; p.B = B; p.M = (int)M; p.N = N; p.K = K;
  p.num_groups = 1; p.group_tile_offsets = nullptr; p.max_m_tiles = 0;
  p.epi_kind = EPI_CONSUME;
  p.epi.out_f32 = out_f32; p.epi.ld_f32 = ld_f32;
  p.epi.out_bf16 = reinterpret_cast<__nv_bfloat16*>(out_bf16); p.epi.ld_bf16 = ld_bf16;
  p.epi.residual = residual; p.epi.ld_res = ld_res;
  p.epi.pair_rows = reinterpret_cast<const __nv_bfloat16*>(pair_rows);
  p.epi.pair_gates = pair_gates;
  p.epi.top_k = k;
  p.epi.n_tokens = M;
  return gemm_bf16(p, (cudaStream_t)stream);
}

int dice_consume_rows(const float* residual, const uint16_t* pair_rows, const float* pair_gates,
                      int64_t n, int k, int hp, float* out, uint16_t* out_bf16, void* stream) {
  if (hp % 4 != 0 || k < 0 || residual == nullptr || out == nullptr) return DICE_ERR_CONTRACT;
  if (n == 0) return DICE_OK;
  launch_pdl(consume_rows_kernel, dim3(grid_for(n * (hp / 4), 256)), dim3(256), 0,
             (cudaStream_t)stream, residual, pair_rows, pair_gates, n, k, hp, out,
             reinterpret_cast<__nv_bfloat16*>(out_bf16));
  return launch_ok();
}

int dice_grouped_ffn(const uint16_t* x_perm, int64_t max_rows, const uint16_t* w1_t,
                     const uint16_t* w2_t, int E, int hp, int ep, const int32_t* tile_offsets,
                     uint16_t* hbuf, uint16_t* y, void* stream) {
  if (E < 1 || E > kMaxGroups || hp % 64 != 0 || ep % 64 != 0 || max_rows % kRowTile != 0)
    return DICE_ERR_CONTRACT;
  cudaStream_t s = (cudaStream_t)stream;
  GemmProblem p{};
  p.A = x_perm; p.A_rows = max_rows; p.B = w1_t; p.M = (int)max_rows; p.N = ep; p.K = hp;
  p.num_groups = E; p.group_tile_offsets = tile_offsets; p.max_m_tiles = (int)(max_rows / kRowTile);
  p.epi_kind = EPI_GELU_BF16;
  p.epi.out_bf16 = reinterpret_cast<__nv_bfloat16*>(hbuf); p.epi.ld_bf16 = ep;
  int rc = gemm_bf16(p, s);
  if (rc) return rc;
  GemmProblem q{};
  q.A = hbuf; q.A_rows = max_rows; q.B = w2_t; q.M = (int)max_rows; q.N = hp; q.K = ep;
  q.num_groups = E; q.group_tile_offsets = tile_offsets; q.max_m_tiles = (int)(max_rows / kRowTile);
  q.epi_kind = EPI_STORE_BF16;
  q.epi.out_bf16 = reinterpret_cast<__nv_bfloat16*>(y); q.epi.ld_bf16 = hp;
  return gemm_bf16(q, s);
}

int dice_cache_assemble(const uint16_t* y, const int32_t* pos, const uint8_t* active,
                        const uint8_t* write, const float* gates, const int32_t* ids, int64_t n, int k,
                        int hp, uint16_t* cache_rows, float* cache_gates, int32_t* cache_ids,
                        float* routed, float* rows_out, float* gates_out, void* stream) {
  if (hp % 64 != 0 || k < 1 || k > 8) return DICE_ERR_CONTRACT;
  if (n == 0) return DICE_OK;
  // register footprint scales with the slot count: instantiate the small k's
  const int grid = grid_for(n * 32, 256);
  cudaStream_t st = (cudaStream_t)stream;
#define DICE_ASM(KK)                                                                           \
  launch_pdl(cache_assemble_kernel<KK>, dim3(grid), dim3(256), 0, st, y, pos, active, write, gates, ids, n, k, hp, \
                                                  cache_rows, cache_gates, cache_ids, routed,  \
                                                  rows_out, gates_out)
  if (k == 1) DICE_ASM(1);
  else if (k == 2) DICE_ASM(2);
  else if (k <= 4) DICE_ASM(4);
  else DICE_ASM(8);
#undef DICE_ASM
  return launch_ok();
}

int dice_gemm(int epi, const uint16_t* A, int64_t M, const uint16_t* B, int N, int K, float* out_f32,
              int64_t ld_f32, uint16_t* out_bf16, int64_t ld_bf16, const float* residual,
              int64_t ld_res, void* stream) {
  if (M < 0 || M > INT_MAX) return DICE_ERR_CONTRACT;
  if (M == 0) return DICE_OK;
  GemmProblem p{};
  p.A = A; p.A_rows = M; p.B = B; p.M = (int)M; p.N = N; p.K = K;
  p.num_groups = 1; p.group_tile_offsets = nullptr; p.max_m_tiles = 0;
  p.epi_kind = epi;
  p.epi.out_f32 = out_f32; p.epi.ld_f32 = ld_f32;
  p.epi.out_bf16 = reinterpret_cast<__nv_bfloat16*>(out_bf16); p.epi.ld_bf16 = ld_bf16;
  p.epi.residual = residual; p.epi.ld_res = ld_res;
  if (epi < EPI_STORE_BF16 || epi > EPI_GELU_RESID) return DICE_ERR_CONTRACT;   // public kinds only
  if (epi == EPI_GELU_RESID && residual == nullptr) return DICE_ERR_CONTRACT;
  return gemm_bf16(p, (cudaStream_t)stream);
}

int dice_combine(const float* base, const float* rows, const float* gates, const float* residual,
                 int64_t n, int k, int hp, float* out, uint16_t* out_bf16, void* stream) {
  if (hp % 4 != 0) return DICE_ERR_CONTRACT;
  if (n == 0) return DICE_OK;
  launch_pdl(combine_kernel, dim3(grid_for(n * (hp / 4), 256)), dim3(256), 0, (cudaStream_t)stream, 
      base, rows, gates, residual, n, k, hp, out, reinterpret_cast<__nv_bfloat16*>(out_bf16));
  return launch_ok();
}

int dice_denoise(float* x, uint16_t* x16, const float* y, float eta, int64_t n, int hp,
                 int32_t* status, int step, void* stream) {
  if (hp % 4 != 0) return DICE_ERR_CONTRACT;
  const int64_t c4 = n * hp / 4;
  if (c4 == 0) return DICE_OK;
  launch_pdl(denoise_kernel, dim3(grid_for(c4, 256)), dim3(256), 0, (cudaStream_t)stream, 
      x, reinterpret_cast<__nv_bfloat16*>(x16), y, eta, c4, status, step);
  return launch_ok();
}

int dice_pack_rows(const float* in, int64_t n, int cols, int64_t ld_in, int hp, float* out32,
                   uint16_t* out16, void* stream) {
  if (cols > hp) return DICE_ERR_CONTRACT;
  if (n == 0) return DICE_OK;
  pack_rows_kernel<<<grid_for(n * hp, 256), 256, 0, (cudaStream_t)stream>>>(
      in, n, cols, ld_in, hp, out32, reinterpret_cast<__nv_bfloat16*>(out16));
  return launch_ok();
}

int64_t dice_similarity_partial_words(void) { return 4 * (int64_t)kSimBlocks; }

int dice_step_similarity(float* prev, const float* cur, int64_t n, int cols, int64_t ld_prev,
                         int64_t ld_cur, int32_t* prev_top, int64_t top_stride,
                         const int32_t* cur_ids, int k, int roll, double* partials, double* out,
                         void* stream) {
  if (n < 0 || cols < 0 || k < 1 || cols > ld_prev || cols > ld_cur) return DICE_ERR_CONTRACT;
  if (out == nullptr || partials == nullptr) return DICE_ERR_CONTRACT;
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0)
    return cudaMemsetAsync(out, 0, 4 * sizeof(double), s) == cudaSuccess ? DICE_OK : DICE_ERR_CUDA;
  if (prev == nullptr || cur == nullptr || prev_top == nullptr || cur_ids == nullptr)
    return DICE_ERR_CONTRACT;
  launch_pdl(similarity_partial_kernel, dim3(kSimBlocks), dim3(kSimThreads), 0, s, prev, cur, n,
             cols, ld_prev, ld_cur, prev_top, top_stride, cur_ids, k, roll, partials);
  launch_pdl(similarity_final_kernel, dim3(1), dim3(kSimThreads), 0, s,
             (const double*)partials, kSimBlocks, out);
  return launch_ok();
}

}  // extern "C"
