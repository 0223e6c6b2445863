// Warp-specialised tcgen05 GEMM for sm_100a: C[M,N] = A[M,K] * B[N,K]^T
// (both operands K-major bf16, fp32 accumulation in TMEM), persistent over
// 256 x BN output tiles computed by CTA pairs (cta_group::2), TMA-fed
// multi-stage smem ring, double-buffered TMEM accumulators so the epilogue of
// tile i overlaps the MMAs of tile i+1.
//
// One kernel serves every dense contraction of the MoE layer:
//   * grouped expert FFN (expert_forward, model.py:226-232): rows of A are the
//     expert-sorted token rows padded per expert to 256-row tiles; B is the
//     stacked per-expert weight [G*N, K]; a device-resident tile->expert prefix
//     (group_tile_offsets) selects the B block per tile, so no host sync.
//   * shared FFN (shared_forward, model.py:235-241) with the S shared experts
//     concatenated along N (GEMM1) / K (GEMM2).
//   * mixing block (local_block, model.py:244-252).
// Epilogues fuse exact-erf GELU, the residual add of local_block, the expert
// rows' store into the layer's pair rows (TokenCache rows, policies.py:188-208)
// and the consume step u + (shared + sum_s g_s row_s) (schedules.py:308-317,
// model.py:279-298) that reads them back.
#include "dice_gemm.h"
#include "dice_ptx.cuh"

#include <climits>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

namespace dice {

constexpr int BM = 128;
constexpr int BK = 64;       // 64 bf16 = 128 B = one swizzle row
constexpr int UMMA_K = 16;
constexpr int kEpiWarps = 12;   // 3 per TMEM lane quadrant
constexpr int kEpiGroups = kEpiWarps / 4;
constexpr int kThreads = 128 + 32 * kEpiWarps;  // w0 TMA, w1 MMA, w2 TMEM alloc, w3 idle, w4.. epilogue

constexpr int kMaxStages = 12;

struct __align__(8) GemmShared {
  uint64_t full[kMaxStages];
  uint64_t empty[kMaxStages];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint32_t tmem_base;
  int m_tiles;
  int group_off[kMaxGroups + 1];
};

__device__ __forceinline__ int find_group(const int* off, int groups, int m_tile) {
  int g = 0;
  while (g + 1 < groups && off[g + 1] <= m_tile) ++g;
  return g;
}

// Epilogue on 4 consecutive columns per lane: 8 lanes cover the 32 columns of
// one output row, a warp covers 4 rows per pass, so residual loads and f32 /
// bf16 stores are coalesced 128-byte / 64-byte row segments. All passes'
// global loads are issued before any math so their latencies overlap.
__device__ __forceinline__ float4 bf16x4_to_f32(uint2 w) {
  return make_float4(__uint_as_float(w.x << 16), __uint_as_float(w.x & 0xFFFF0000u),
                     __uint_as_float(w.y << 16), __uint_as_float(w.y & 0xFFFF0000u));
}
__device__ __forceinline__ float4 add_scaled(float4 x, float g, float4 r) {
  // x + g * r with the product and the sum each rounded (combine_outputs,
  // model.py:295-297: out += gates[:, s] * rows[s])
  return make_float4(__fadd_rn(x.x, __fmul_rn(g, r.x)), __fadd_rn(x.y, __fmul_rn(g, r.y)),
                     __fadd_rn(x.z, __fmul_rn(g, r.z)), __fadd_rn(x.w, __fmul_rn(g, r.w)));
}

template <int EPI>
__device__ __forceinline__ void epilogue_chunk(const GemmArgs& a, float* stage, int lane,
                                               int row0, int row_limit, int col0) {
  const int q = lane & 7;
  const int col = col0 + 4 * q;
  constexpr int KF = 2;   // consume: routed slots prefetched with the residual (more: in turn)
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    float4 v[4], r[4];
    uint2 pr[KF][4];
    float pg[KF][4];
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int rr = (half * 4 + it) * 4 + (lane >> 3);
      v[it] = *reinterpret_cast<const float4*>(stage + rr * 32 + ((q ^ (rr & 7)) << 2));
    }
    if constexpr (EPI == EPI_GELU_RESID || EPI == EPI_CONSUME) {
#pragma unroll
      for (int it = 0; it < 4; ++it) {
        const int64_t row = row0 + (half * 4 + it) * 4 + (lane >> 3);
        if (row < row_limit) {
          r[it] = __ldg(reinterpret_cast<const float4*>(a.residual + row * a.ld_res + col));
          if constexpr (EPI == EPI_CONSUME) {
#pragma unroll
            for (int s = 0; s < KF; ++s) {
              if (s < a.top_k) {
                pr[s][it] = __ldg(reinterpret_cast<const uint2*>(
                    a.pair_rows + ((int64_t)s * a.n_tokens + row) * a.N + col));
                pg[s][it] = __ldg(a.pair_gates + row * a.top_k + s);
              }
            }
          }
        }
      }
    }
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int64_t row = row0 + (half * 4 + it) * 4 + (lane >> 3);
      float4 x = v[it];
      if constexpr (EPI == EPI_GELU_BF16 || EPI == EPI_GELU_RESID) {
        const float2 lo = gelu_erf2(make_float2(x.x, x.y));
        const float2 hi = gelu_erf2(make_float2(x.z, x.w));
        x = make_float4(lo.x, lo.y, hi.x, hi.y);
      }
      if constexpr (EPI == EPI_GELU_RESID) {
        x.x += r[it].x; x.y += r[it].y; x.z += r[it].z; x.w += r[it].w;
      }
      if constexpr (EPI == EPI_CONSUME) {
        if (row < row_limit) {
#pragma unroll
          for (int s = 0; s < KF; ++s)
            if (s < a.top_k) x = add_scaled(x, pg[s][it], bf16x4_to_f32(pr[s][it]));
          for (int s = KF; s < a.top_k; ++s) {
            const uint2 w = __ldg(reinterpret_cast<const uint2*>(
                a.pair_rows + ((int64_t)s * a.n_tokens + row) * a.N + col));
            x = add_scaled(x, __ldg(a.pair_gates + row * a.top_k + s), bf16x4_to_f32(w));
          }
          x = make_float4(__fadd_rn(r[it].x, x.x), __fadd_rn(r[it].y, x.y),
                          __fadd_rn(r[it].z, x.z), __fadd_rn(r[it].w, x.w));
        }
      }
      if (row < row_limit) {
        if (a.out_f32 != nullptr) *reinterpret_cast<float4*>(a.out_f32 + row * a.ld_f32 + col) = x;
        if (a.out_bf16 != nullptr) {
          __nv_bfloat162 lo = __floats2bfloat162_rn(x.x, x.y), hi = __floats2bfloat162_rn(x.z, x.w);
          *reinterpret_cast<uint2*>(a.out_bf16 + row * a.ld_bf16 + col) =
              make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
        }
      }
    }
  }
}

// Residual prefetch for the local_block epilogue: the lane's 8 rows x 4 columns
// of the chunk land by cp.async in the same XOR-swizzled 32x32 layout as the
// accumulator staging tile (zero-filled past the last row).
__device__ __forceinline__ void resid_prefetch(const GemmArgs& a, float* rbuf, int lane, int row0,
                                               int row_limit, int col0) {
  const int q = lane & 7;
  const int col = col0 + 4 * q;
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const int rr = it * 4 + (lane >> 3);
    const int64_t row = row0 + rr;
    const bool ok = row < row_limit;
    const float* src = a.residual + (ok ? row : 0) * a.ld_res + col;
    const uint32_t dst = smem_u32(rbuf + rr * 32 + ((q ^ (rr & 7)) << 2));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
                 "r"(ok ? 16 : 0) : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

__device__ __forceinline__ void resid_wait() {
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncwarp();
}

// GELU_RESID epilogue with the residual already in smem (rbuf); when `next_col0`
// is valid the next chunk's residual prefetch is issued once this chunk's has
// been read into registers.
__device__ __forceinline__ void epilogue_gelu_resid_pf(const GemmArgs& a, const float* stage,
                                                       float* rbuf, int lane, int row0,
                                                       int row_limit, int col0, int next_col0) {
  const int q = lane & 7;
  const int col = col0 + 4 * q;
  float4 r[8];
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const int rr = it * 4 + (lane >> 3);
    r[it] = *reinterpret_cast<const float4*>(rbuf + rr * 32 + ((q ^ (rr & 7)) << 2));
  }
  __syncwarp();
  if (next_col0 >= 0) resid_prefetch(a, rbuf, lane, row0, row_limit, next_col0);
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const int rr = it * 4 + (lane >> 3);
    const float4 v = *reinterpret_cast<const float4*>(stage + rr * 32 + ((q ^ (rr & 7)) << 2));
    const float2 lo = gelu_erf2(make_float2(v.x, v.y));
    const float2 hi = gelu_erf2(make_float2(v.z, v.w));
    const float4 x = make_float4(lo.x + r[it].x, lo.y + r[it].y, hi.x + r[it].z, hi.y + r[it].w);
    const int64_t row = row0 + rr;
    if (row < row_limit) {
      if (a.out_f32 != nullptr) *reinterpret_cast<float4*>(a.out_f32 + row * a.ld_f32 + col) = x;
      if (a.out_bf16 != nullptr) {
        __nv_bfloat162 l2 = __floats2bfloat162_rn(x.x, x.y), h2 = __floats2bfloat162_rn(x.z, x.w);
        *reinterpret_cast<uint2*>(a.out_bf16 + row * a.ld_bf16 + col) =
            make_uint2(*reinterpret_cast<uint32_t*>(&l2), *reinterpret_cast<uint32_t*>(&h2));
      }
    }
  }
}

// --------------------------------------------------------- CTA-pair kernel
// cta_group::2: a cluster of two CTAs computes a 256 x BN tile. Each CTA
// stages its own 128 rows of A and half (BN/2 rows) of B, so per-CTA operand
// traffic per MMA FLOP is 2/3 of the single-CTA 128 x BN tile; the even CTA
// issues the pair MMAs and both CTAs drain their 128 TMEM lanes. TMEM holds
// two BN-column accumulators, so the epilogue of tile i overlaps the MMAs of
// tile i + 1.
template <int BN, bool DIRECT, bool RESID_PF = false>
struct PairCfg {
  static constexpr int kTN = BN;
  static constexpr int kAccBufs = 2;
  static constexpr int kABytes = BM * BK * 2;
  static constexpr int kBBytes = (BN / 2) * BK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  // bf16-only epilogues store straight from registers (64 contiguous bytes of
  // one row per lane, whole sectors), so their smem goes to the operand ring
  // RESID_PF (the local_block GELU_RESID epilogue): a second 32x32 f32 tile per
  // epilogue warp receives the chunk's residual by cp.async ahead of its use
  static constexpr int kEpiBytes = DIRECT ? 0 : kEpiWarps * 32 * 32 * 4 * (RESID_PF ? 2 : 1);
  static constexpr int kBudget = 232448 - kEpiBytes - 2048;
  static constexpr int kStages = kBudget / kStageBytes > kMaxStages ? kMaxStages : kBudget / kStageBytes;
  static constexpr int kTmemCols = kAccBufs * kTN <= 256 ? 256 : 512;
  static_assert(kAccBufs * kTN <= 512, "TMEM holds 512 fp32 columns");
  static constexpr int kSmemBytes = kStages * kStageBytes + kEpiBytes + 2048;
};

// Direct bf16 epilogue: this lane owns one row and 32 consecutive columns.
template <int EPI>
__device__ __forceinline__ void epilogue_direct(const GemmArgs& a, const uint32_t (&r)[32],
                                                int64_t row, int col0, int64_t pair_row) {
  uint32_t w[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    float2 v = make_float2(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1]));
    if constexpr (EPI == EPI_GELU_BF16) v = gelu_erf2(v);
    __nv_bfloat162 b = __floats2bfloat162_rn(v.x, v.y);
    w[j] = *reinterpret_cast<uint32_t*>(&b);
  }
  __nv_bfloat16* out = a.out_bf16 + row * a.ld_bf16;
  if constexpr (EPI == EPI_STORE_PAIR) {
    // (token, slot) pair of this expert row -> the layer's pair rows [s][t]
    const int p = a.row_pair[pair_row];
    if (p < 0) return;                       // padding row of an expert group
    const int64_t t = p / a.top_k;
    const int s = p - (int)t * a.top_k;
    out = a.out_bf16 + ((int64_t)s * a.n_tokens + t) * a.ld_bf16;
    if (col0 == 0) {
      if (a.cache_gates != nullptr) a.cache_gates[p] = a.pair_gates[p];
      if (a.cache_ids != nullptr) a.cache_ids[p] = a.pair_ids[p];
    }
  }
  if constexpr (EPI == EPI_STORE_SCATTER) {
    const int i = a.row_pair[row];
    if (i < 0) return;                       // padding row of an expert group
    const int src = (int)(i / a.scatter_cap);
    const int4 m = reinterpret_cast<const int4*>(a.scatter_meta)[i];   // {e_local, pair, gate, expert}
    const int64_t t = m.y / a.top_k;
    const int s = m.y - (int)t * a.top_k;
    out = reinterpret_cast<__nv_bfloat16*>(a.scatter_rows[src]) +
          ((int64_t)s * a.scatter_n[src] + t) * a.ld_bf16;
    if (col0 == 0) {
      reinterpret_cast<float*>(a.scatter_gates[src])[m.y] = __int_as_float(m.z);
      reinterpret_cast<int32_t*>(a.scatter_ids[src])[m.y] = m.w;
    }
  }
  uint4* dst = reinterpret_cast<uint4*>(out + col0);
#pragma unroll
  for (int j = 0; j < 4; ++j) dst[j] = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
}

// MC = 2: a cluster of two CTA pairs computes the n-blocks 2j, 2j + 1 of one
// m-tile; each CTA loads half of the A block both pairs need and TMA-multicasts
// it to its counterpart in the other pair (L2 reads of A halve), and a ring
// slot is refilled only after both pairs' MMAs have read it.
template <int BN, int EPI, bool DIRECT, int MC>
__global__ void __launch_bounds__(kThreads, 1)
gemm_bf16_pair(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const GemmArgs args, const __grid_constant__ CUtensorMap tmA2,
               const __grid_constant__ CUtensorMap tmB2, const GemmArgs args2) {
  // args2.num_m_tiles > 0: a second, dense problem with the same K and epilogue
  // kind runs in the same persistent launch; its tiles follow the first's
  // (one launch and one wave tail for two independent GEMMs)
  constexpr bool kResidPF = EPI == EPI_GELU_RESID;
  using C = PairCfg<BN, DIRECT, kResidPF>;
  constexpr int TN = C::kTN;
  const int kStages = args.stages;   // <= C::kStages (host-clamped)
  constexpr int kPairM = 2 * BM;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smA = smem;
  uint8_t* smB = smem + C::kStages * C::kABytes;
  float* sm_epi = reinterpret_cast<float*>(smem + C::kStages * C::kStageBytes);
  GemmShared* sh = reinterpret_cast<GemmShared*>(smem + C::kStages * C::kStageBytes + C::kEpiBytes);

  static_assert(MC == 1 || MC == 2, "one or two CTA pairs per cluster");
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  const uint32_t rank = crank & 1;           // CTA within its pair
  const uint32_t pp = crank >> 1;            // pair within the cluster
  const uint32_t leader = crank & ~1u;       // the pair's even CTA

  // prologue before the programmatic-dependency wait: it touches no memory the
  // stream predecessor writes, so under PDL it overlaps that kernel's tail
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) { mbar_init(&sh->full[s], 2); mbar_init(&sh->empty[s], MC); }
    for (int b = 0; b < 2; ++b) { mbar_init(&sh->tfull[b], 1); mbar_init(&sh->tempty[b], 2 * kEpiWarps); }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA); tma_prefetch_desc(&tmB);
    if (args2.num_m_tiles > 0) { tma_prefetch_desc(&tmA2); tma_prefetch_desc(&tmB2); }
  }
  if (warp == 2) tmem_alloc_pair<C::kTmemCols>(&sh->tmem_base);
  pdl_wait();
  if (threadIdx.x == 0) {
    if (args.group_tile_offsets != nullptr) {
      for (int g = 0; g <= args.num_groups; ++g) sh->group_off[g] = args.group_tile_offsets[g];
      sh->m_tiles = sh->group_off[args.num_groups];
    } else {
      sh->group_off[0] = 0;
      sh->group_off[1] = args.num_m_tiles;
      sh->m_tiles = args.num_m_tiles;
    }
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  pdl_trigger();

  const uint32_t tmem_base = sh->tmem_base;
  const int m_tiles = sh->m_tiles;  // 256-row tiles
  const int groups = args.group_tile_offsets != nullptr ? args.num_groups : 1;
  const int n_blocks = args.num_n_blocks;
  const int k_blocks = args.num_k_blocks;
  // work items: (m tile, MC consecutive n blocks), one n block per pair
  const int n_units = n_blocks / MC;
  const int T1 = m_tiles * n_units;
  const int n_units2 = args2.num_n_blocks / MC;
  const int num_tiles = T1 + (args2.num_m_tiles > 0 ? args2.num_m_tiles * n_units2 : 0);
  // item -> (problem, n block, m tile); N-fastest within each problem
  auto locate = [&](int tile, int& prob, int& n_blk, int& m_tile) {
    if (tile < T1) { prob = 0; n_blk = (tile % n_units) * MC + pp; m_tile = tile / n_units; }
    else {
      prob = 1; const int t2 = tile - T1;
      n_blk = (t2 % n_units2) * MC + pp; m_tile = t2 / n_units2;
    }
  };
  const int pair = blockIdx.x / (2 * MC);         // cluster index
  const int num_pairs = gridDim.x / (2 * MC);
  const int n_items = pair < num_tiles ? (num_tiles - 1 - pair) / num_pairs + 1 : 0;

  // producer (warp 0) and MMA issuer (warp 1 of the even CTA): converged
  // loops, one elected lane issues (elect_one)
  if (warp == 0) {
    {
      int stage = 0;
      uint32_t phase = 0;
      for (int it = 0; it < n_items; ++it) {
        // the dual launch (expert + shared GEMM1) runs its items last to first:
        // the grouped expert tiles, whose hbuf the next launch (the expert GEMM2)
        // reads first-to-last, are written last and are still in L2 when it
        // starts (+0.2 % img/s over forward order in three same-box pairs, +0.2 %
        // more over reversing every launch)
        const int xi = pair + it * num_pairs;
        const int tile = args2.num_m_tiles > 0 ? num_tiles - 1 - xi : xi, k0 = 0, k1 = k_blocks;
        int prob, n_blk, m_tile;   // N-fastest: resident tiles share A rows
        locate(tile, prob, n_blk, m_tile);
        const int g = prob == 0 ? find_group(sh->group_off, groups, m_tile) : 0;
        const int a_row = (prob == 0 && args.a_group_stride > 0)
                              ? (int)(g * args.a_group_stride) +
                                    (m_tile - sh->group_off[g]) * kPairM + rank * BM
                              : m_tile * kPairM + rank * BM;
        const int b_row = g * (prob == 0 ? args.N : args2.N) + n_blk * TN + rank * (BN / 2);
        const CUtensorMap* mA = prob == 0 ? &tmA : &tmA2;
        const CUtensorMap* mB = prob == 0 ? &tmB : &tmB2;
        for (int kb = k0; kb < k1; ++kb) {
          mbar_wait(&sh->empty[stage], phase ^ 1);
          if (elect_one()) {
            mbar_arrive_expect_tx_cluster(mapa_shared(smem_u32(&sh->full[stage]), leader),
                                          C::kStageBytes);
            if constexpr (MC == 1) {
              tma_load_2d_pair(smA + stage * C::kABytes, mA, &sh->full[stage], kb * BK, a_row);
            } else {   // this CTA's half of the A block, to itself and its counterpart
              tma_load_2d_pair_mc(smA + stage * C::kABytes + pp * (BM / 2) * BK * 2, mA,
                                  &sh->full[stage], kb * BK, a_row + (int)pp * (BM / 2),
                                  (uint16_t)((1u << rank) | (1u << (2 + rank))));
            }
            tma_load_2d_pair(smB + stage * C::kBBytes, mB, &sh->full[stage], kb * BK, b_row);
          }
          __syncwarp();
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(kPairM, BN);
      int stage = 0;
      uint32_t phase = 0;
      for (int local = 0; local < n_items; ++local) {
        const int k0 = 0, k1 = k_blocks;
        const int acc = C::kAccBufs == 2 ? (local & 1) : 0;
        const uint32_t acc_phase = C::kAccBufs == 2 ? ((local >> 1) & 1) : (local & 1);
        mbar_wait(&sh->tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * TN;
        for (int kb = k0; kb < k1; ++kb) {
          mbar_wait(&sh->full[stage], phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(smA + stage * C::kABytes);
          const uint32_t b_base = smem_u32(smB + stage * C::kBBytes);
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < BK / UMMA_K; ++k) {
              umma_bf16_pair(d_tmem, umma_desc_sw128(a_base + k * UMMA_K * 2),
                             umma_desc_sw128(b_base + k * UMMA_K * 2), idesc,
                             (kb != k0 || k != 0) ? 1u : 0u);
            }
            umma_commit_pair(&sh->empty[stage], MC == 1 ? (uint16_t)0x3 : (uint16_t)0xF);
          }
          __syncwarp();
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) umma_commit_pair(&sh->tfull[acc], (uint16_t)(0x3u << (2 * pp)));
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    const int sub = warp & 3;
    const int grp = (warp - 4) >> 2;
    float* stage = sm_epi + (warp - 4) * 1024;
    float* rbuf = sm_epi + kEpiWarps * 1024 + (warp - 4) * 1024;   // (kResidPF only)
    const int row_limit = args.group_tile_offsets != nullptr ? INT_MAX : args.M_valid;
    const uint32_t tempty_leader0 = mapa_shared(smem_u32(&sh->tempty[0]), leader);
    const uint32_t tempty_leader1 = mapa_shared(smem_u32(&sh->tempty[1]), leader);
    for (int local = 0; local < n_items; ++local) {
      const int xl = pair + local * num_pairs;                        // as the producer
      const int tile = args2.num_m_tiles > 0 ? num_tiles - 1 - xl : xl;
      int prob, n_blk, m_tile;
      locate(tile, prob, n_blk, m_tile);
      const GemmArgs& ar = prob == 0 ? args : args2;
      const int rl = prob == 0 ? row_limit : args2.M_valid;
      const int acc = C::kAccBufs == 2 ? (local & 1) : 0;
      const uint32_t acc_phase = C::kAccBufs == 2 ? ((local >> 1) & 1) : (local & 1);
      const int row0 = m_tile * kPairM + rank * BM + sub * 32;
      // STORE_PAIR over capacity-strided expert regions: the row -> pair map
      // entry of this lane's row
      int64_t pair_row0 = row0;
      if constexpr (EPI == EPI_STORE_PAIR) {
        if (ar.pair_group_stride > 0) {
          const int g = find_group(sh->group_off, groups, m_tile);
          pair_row0 = g * ar.pair_group_stride + (int64_t)(m_tile - sh->group_off[g]) * kPairM +
                      rank * BM + sub * 32;
        }
      }
      if constexpr (kResidPF) {   // first chunk's residual while the MMAs run
        if (grp * 32 < TN && n_blk * TN + grp * 32 < ar.N)
          resid_prefetch(ar, rbuf, lane, row0, rl, n_blk * TN + grp * 32);
      }
      mbar_wait(&sh->tfull[acc], acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (int ci = grp; ci < TN / 32; ci += kEpiGroups) {
        const int col_in_tile = ci * 32;
        const int col0 = n_blk * TN + col_in_tile;
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(sub * 32) << 16) + acc * TN + col_in_tile, r);
        tmem_ld_wait();
        if (col0 >= ar.N) continue;  // warp-uniform
        if constexpr (DIRECT) {
          const int64_t row = row0 + lane;
          if (row < rl) epilogue_direct<EPI>(ar, r, row, col0, pair_row0 + lane);
          continue;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
          *reinterpret_cast<float4*>(stage + lane * 32 + ((q ^ (lane & 7)) << 2)) =
              make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                          __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
        __syncwarp();
        if constexpr (kResidPF) {
          resid_wait();
          const int nci = ci + kEpiGroups;
          const int ncol = n_blk * TN + nci * 32;
          epilogue_gelu_resid_pf(ar, stage, rbuf, lane, row0, rl, col0,
                                 (nci < TN / 32 && ncol < ar.N) ? ncol : -1);
        } else {
          epilogue_chunk<EPI>(ar, stage, lane, row0, rl, col0);
        }
        __syncwarp();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(acc ? tempty_leader1 : tempty_leader0);
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair<C::kTmemCols>(tmem_base);
  }
}

// ------------------------------------------------------------------- host
namespace {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

struct MapKey {
  const void* ptr; int64_t rows, cols; int box_rows;
  bool operator==(const MapKey& o) const {
    return ptr == o.ptr && rows == o.rows && cols == o.cols && box_rows == o.box_rows;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    return std::hash<const void*>()(k.ptr) ^ (std::hash<int64_t>()(k.rows) * 31) ^
           (std::hash<int64_t>()(k.cols) * 131) ^ (size_t)k.box_rows;
  }
};

std::mutex g_map_mu;
std::unordered_map<MapKey, CUtensorMap, MapKeyHash> g_maps;

// Row-major bf16 [rows, cols] with a (BK x box_rows) box and 128-byte swizzle.
int tensor_map(const void* ptr, int64_t rows, int64_t cols, int box_rows, CUtensorMap* out) {
  MapKey key{ptr, rows, cols, box_rows};
  {
    std::lock_guard<std::mutex> lk(g_map_mu);
    auto it = g_maps.find(key);
    if (it != g_maps.end()) { *out = it->second; return 0; }
  }
  EncodeTiledFn fn = encode_fn();
  if (fn == nullptr) return DICE_ERR_CUDA;
  if ((cols * 2) % 16 != 0 || (reinterpret_cast<uintptr_t>(ptr) & 15) != 0) return DICE_ERR_CONTRACT;
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(cols * 2)};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box,
                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return DICE_ERR_CUDA;
  std::lock_guard<std::mutex> lk(g_map_mu);
  if (g_maps.size() > 4096) g_maps.clear();
  g_maps[key] = m;
  *out = m;
  return 0;
}

int num_sms() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

// MC: CTA pairs per cluster (2: A multicast across the two pairs of an m-tile;
// the A tensor map's box is then BM / 2 rows and the n-block counts are even)
template <int BN, int EPI, bool DIRECT, int MC = 1>
int launch_pair(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& a, int max_tiles,
                cudaStream_t stream, const CUtensorMap* ta2 = nullptr,
                const CUtensorMap* tb2 = nullptr, const GemmArgs* a2 = nullptr) {
  using C = PairCfg<BN, DIRECT, EPI == EPI_GELU_RESID>;
  auto kern = gemm_bf16_pair<BN, EPI, DIRECT, MC>;
  constexpr int CL = 2 * MC;               // CTAs per cluster
  static int max_clusters = -1;
  if (max_clusters < 0) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes) !=
        cudaSuccess)
      return DICE_ERR_CUDA;
    // clusters must fit a GPC: a persistent grid larger than the co-resident
    // cluster count would run its last clusters as a second wave
    cudaLaunchConfig_t q = {};
    q.gridDim = dim3(num_sms() - num_sms() % CL);
    q.blockDim = dim3(kThreads);
    q.dynamicSmemBytes = C::kSmemBytes;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    q.attrs = at;
    q.numAttrs = 1;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, kern, &q) != cudaSuccess || nc <= 0) {
      cudaGetLastError();
      nc = num_sms() / CL;
    }
    max_clusters = nc;
  }
  if (a.num_n_blocks % MC != 0 || (a2 != nullptr && a2->num_n_blocks % MC != 0))
    return DICE_ERR_CONTRACT;
  const int items = (max_tiles + (a2 != nullptr ? a2->num_m_tiles * a2->num_n_blocks : 0)) / MC;
  int grid = items < max_clusters ? CL * items : CL * max_clusters;
  if (grid <= 0) return 0;
  GemmArgs aa = a;
  aa.stages = C::kStages;
  GemmArgs bb{};
  if (a2 != nullptr) bb = *a2;
  launch_pdl_cluster(kern, dim3(grid), dim3(kThreads), C::kSmemBytes, stream, CL, ta, tb, aa,
                     a2 != nullptr ? *ta2 : ta, a2 != nullptr ? *tb2 : tb, bb);
  return cudaGetLastError() == cudaSuccess ? 0 : DICE_ERR_CUDA;
}

template <int BN, int MC = 1>
int dispatch_pair(int epi, const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& a,
                  int max_tiles, cudaStream_t s) {
  switch (epi) {
    case EPI_STORE_BF16: return launch_pair<BN, EPI_STORE_BF16, true, MC>(ta, tb, a, max_tiles, s);
    case EPI_GELU_BF16: return launch_pair<BN, EPI_GELU_BF16, true, MC>(ta, tb, a, max_tiles, s);
    case EPI_STORE_PAIR: return launch_pair<BN, EPI_STORE_PAIR, true, MC>(ta, tb, a, max_tiles, s);
    case EPI_STORE_SCATTER: return launch_pair<BN, EPI_STORE_SCATTER, true, MC>(ta, tb, a, max_tiles, s);
    case EPI_STORE_F32: return launch_pair<BN, EPI_STORE_F32, false, MC>(ta, tb, a, max_tiles, s);
    case EPI_GELU_RESID: return launch_pair<BN, EPI_GELU_RESID, false, MC>(ta, tb, a, max_tiles, s);
    case EPI_CONSUME: return launch_pair<BN, EPI_CONSUME, false, MC>(ta, tb, a, max_tiles, s);
    default: return DICE_ERR_CONTRACT;
  }
}

}  // namespace

struct TileChoice {
  int bn;        // MMA N per accumulator = output columns per tile
  int tile_n;
  int mc;        // CTA pairs per cluster sharing the A block
};

// Every GEMM runs on the CTA-pair kernel (256-row tiles: the permute pads
// expert groups to 256 rows) with two TMEM accumulators. Tile width: 256 when
// N allows, else 192 / 128. (256 x 384 tiles of two accumulators sharing each
// staged A block won while the MMA issue was the bottleneck; with the
// converged issue loop the double-buffered 256 x 192 tile is faster at
// N = 1152: 1452 vs 1370 TF/s at 16384 x 1152 x 4608.)
TileChoice choose_tile(const GemmProblem& p) {
  TileChoice c{};
  c.bn = (p.N % 256 == 0) ? 256 : (p.N % 192 == 0 ? 192 : 128);
  c.tile_n = c.bn;
  // N = 1152-class GEMMs (256 x 192 tiles, an even number of n-blocks): clusters
  // of two CTA pairs share each A block by TMA multicast. Only 33 clusters of
  // four fit the GPCs (132 of 148 SMs), but halving the A reads from L2 cuts
  // enough energy that the power-capped step runs ~5 % higher clocks: +0.8 %
  // img/s in-step (35.0-35.2 vs 34.8, same box); for the 256 x 256 GEMM1s the
  // lost SMs weigh more (1370 vs 1477 TF/s) and they stay on pairs
  c.mc = (c.bn == 192 && ((p.N + c.tile_n - 1) / c.tile_n) % 2 == 0) ? 2 : 1;
  return c;
}

namespace {
// tensor maps + kernel arguments of one problem for its tile choice
int prepare(const GemmProblem& p, const TileChoice& tc, CUtensorMap* ta, CUtensorMap* tb,
            GemmArgs* a) {
  if (p.K <= 0 || p.N <= 0 || p.N % 32 != 0 || p.K % 8 != 0) return DICE_ERR_CONTRACT;
  if (p.num_groups < 1 || p.num_groups > kMaxGroups) return DICE_ERR_CONTRACT;
  const int tile_m = 2 * BM;
  int rc = tensor_map(p.A, p.A_rows, p.K, BM / tc.mc, ta);
  if (rc) return rc;
  rc = tensor_map(p.B, (int64_t)p.num_groups * p.N, p.K, tc.bn / 2, tb);
  if (rc) return rc;
  *a = p.epi;
  a->M_valid = p.M;
  a->N = p.N;
  a->K = p.K;
  a->num_n_blocks = (p.N + tc.tile_n - 1) / tc.tile_n;
  a->num_k_blocks = (p.K + BK - 1) / BK;
  a->group_tile_offsets = p.group_tile_offsets;
  a->num_groups = p.num_groups;
  a->num_m_tiles = p.group_tile_offsets != nullptr ? p.max_m_tiles : (p.M + tile_m - 1) / tile_m;
  return 0;
}
}  // namespace

int gemm_bf16(const GemmProblem& p, cudaStream_t stream) {
  const TileChoice tc = choose_tile(p);
  const int bn = tc.bn;
  CUtensorMap ta, tb;
  GemmArgs a;
  int rc = prepare(p, tc, &ta, &tb, &a);
  if (rc) return rc;
  const int max_tiles = a.num_m_tiles * a.num_n_blocks;
  if (max_tiles == 0) return 0;
  if (tc.mc == 2) {
    if (bn == 256) return dispatch_pair<256, 2>(p.epi_kind, ta, tb, a, max_tiles, stream);
    if (bn == 192) return dispatch_pair<192, 2>(p.epi_kind, ta, tb, a, max_tiles, stream);
    return dispatch_pair<128, 2>(p.epi_kind, ta, tb, a, max_tiles, stream);
  }
  if (bn == 256) return dispatch_pair<256>(p.epi_kind, ta, tb, a, max_tiles, stream);
  if (bn == 192) return dispatch_pair<192>(p.epi_kind, ta, tb, a, max_tiles, stream);
  return dispatch_pair<128>(p.epi_kind, ta, tb, a, max_tiles, stream);
}

// Two independent GEMMs with the same K and bf16-only epilogue kind in ONE
// persistent launch (p1 may be grouped, p2 dense): the grouped expert GEMM1
// and the shared-expert GEMM1 of a stage. Falls back to two launches when the
// tile choices differ.
int gemm_bf16_dual(const GemmProblem& p1, const GemmProblem& p2, cudaStream_t stream) {
  const TileChoice c1 = choose_tile(p1), c2 = choose_tile(p2);
  const bool ok = p1.K == p2.K && p1.epi_kind == p2.epi_kind &&
                  (p1.epi_kind == EPI_STORE_BF16 || p1.epi_kind == EPI_GELU_BF16) &&
                  p2.group_tile_offsets == nullptr && c1.bn == c2.bn && c1.mc == c2.mc &&
                  (c1.bn == 256 || c1.bn == 192);
  if (!ok) {
    const int rc = gemm_bf16(p1, stream);
    return rc ? rc : gemm_bf16(p2, stream);
  }
  CUtensorMap ta1, tb1, ta2, tb2;
  GemmArgs a1, a2;
  int rc = prepare(p1, c1, &ta1, &tb1, &a1);
  if (rc) return rc;
  rc = prepare(p2, c2, &ta2, &tb2, &a2);
  if (rc) return rc;
  const int t1 = a1.num_m_tiles * a1.num_n_blocks;
  if (a2.num_m_tiles * a2.num_n_blocks == 0) return gemm_bf16(p1, stream);
  if (c1.bn == 256 && c1.mc == 2) {
    return p1.epi_kind == EPI_GELU_BF16
               ? launch_pair<256, EPI_GELU_BF16, true, 2>(ta1, tb1, a1, t1, stream, &ta2, &tb2, &a2)
               : launch_pair<256, EPI_STORE_BF16, true, 2>(ta1, tb1, a1, t1, stream, &ta2, &tb2, &a2);
  }
  if (c1.bn == 256) {
    return p1.epi_kind == EPI_GELU_BF16
               ? launch_pair<256, EPI_GELU_BF16, true>(ta1, tb1, a1, t1, stream, &ta2, &tb2, &a2)
               : launch_pair<256, EPI_STORE_BF16, true>(ta1, tb1, a1, t1, stream, &ta2, &tb2, &a2);
  }
  if (c1.mc == 2) {
    return p1.epi_kind == EPI_GELU_BF16
               ? launch_pair<192, EPI_GELU_BF16, true, 2>(ta1, tb1, a1, t1, stream, &ta2, &tb2, &a2)
               : launch_pair<192, EPI_STORE_BF16, true, 2>(ta1, tb1, a1, t1, stream, &ta2, &tb2, &a2);
  }
  return p1.epi_kind == EPI_GELU_BF16
             ? launch_pair<192, EPI_GELU_BF16, true>(ta1, tb1, a1, t1, stream, &ta2, &tb2, &a2)
             : launch_pair<192, EPI_STORE_BF16, true>(ta1, tb1, a1, t1, stream, &ta2, &tb2, &a2);
}

}  // namespace dice
