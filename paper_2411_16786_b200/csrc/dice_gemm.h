// Internal GEMM interface shared by the C-ABI layer and the kernels.
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "../../include/dice_b200.h"

namespace dice {

constexpr int kMaxGroups = 64;

enum EpiKind : int {
  EPI_STORE_BF16 = 0,  // out_bf16 = acc
  EPI_GELU_BF16 = 1,   // out_bf16 = gelu(acc)
  EPI_STORE_F32 = 2,   // out_f32 = acc (and out_bf16 if set)
  EPI_GELU_RESID = 3,  // v = gelu(acc) + residual -> out_f32, out_bf16   (local_block)
  EPI_CONSUME = 4,     // v = residual + (acc + addend) -> out_f32, out_bf16 (consume)
  // GELU_RESID whose epilogue also emits partial router logits of the finished
  // u rows (gate fused into local_block's GEMM, E = 8 / 16 experts)
  EPI_GELU_RESID_GATE8 = 5,
  EPI_GELU_RESID_GATE16 = 6,
  // expert GEMM2 with the routed combine fused (k <= 2): each output row (a
  // (token, slot) pair) is rounded to bf16 as a fresh expert row, persisted to the
  // token cache when the pair refreshes it, and g * row is added into the
  // token's combine slot (pre-initialised with its cached terms)
  EPI_COMBINE = 7,
  // expert-parallel expert GEMM2 with the combine all-to-all fused: each output
  // row (window entry i = row_pair[r] of source rank i / scatter_cap) is stored
  // as bf16 straight into that rank's combine window (peer memory) at its home
  // pair index scatter_meta[i].y, tile by tile as the GEMM finishes them
  EPI_STORE_SCATTER = 8,
};

template <int EPI>
struct EpiTraits {
  static constexpr int base = EPI;
  static constexpr int gate_e = 0;
};
template <>
struct EpiTraits<EPI_GELU_RESID_GATE8> {
  static constexpr int base = EPI_GELU_RESID;
  static constexpr int gate_e = 8;
};
template <>
struct EpiTraits<EPI_GELU_RESID_GATE16> {
  static constexpr int base = EPI_GELU_RESID;
  static constexpr int gate_e = 16;
};

struct GemmArgs {
  int M_valid;
  int N;
  int K;
  int num_n_blocks;
  int num_k_blocks;
  int num_m_tiles;
  const int* group_tile_offsets;
  int num_groups;
  __nv_bfloat16* out_bf16;
  int64_t ld_bf16;
  float* out_f32;
  int64_t ld_f32;
  const float* residual;
  int64_t ld_res;
  const float* addend;
  int64_t ld_add;
  int stages;            // operand ring depth actually used (pair kernel; set by the host)
  const float* gate_w;   // GATE epilogues: W_gate f32 [N, E] (row c = hidden column c)
  float* gate_part;      // GATE epilogues: partial logits f32 [P, M, E], P = gemm_gate_parts()
  // COMBINE: row -> pair map, per-pair gates / cache-write mask, slot [n, N] f32,
  // cache rows of the layer bf16 [k, n, N]
  const int32_t* row_pair;
  const float* pair_gates;
  const uint8_t* pair_write;
  int top_k;
  int64_t n_tokens;
  float* slot;
  __nv_bfloat16* cache_rows;
  // STORE_SCATTER: window metadata int2 [D * cap] (.y = home pair), entries per
  // source rank, and the D combine-window bases (peer-mapped device pointers)
  const void* scatter_meta;
  int64_t scatter_cap;
  uint64_t scatter_dst[16];
};

struct GemmProblem {
  const void* A;          // bf16 [A_rows, K] row-major
  int64_t A_rows;
  const void* B;          // bf16 [num_groups * N, K] row-major
  int M, N, K;
  int num_groups;
  const int* group_tile_offsets;  // device [num_groups+1] m-tile prefix; null => dense
  int max_m_tiles;                // grouped: upper bound of total m tiles
  int epi_kind;
  GemmArgs epi;                   // only the output/residual fields are read
};

int gemm_bf16(const GemmProblem& p, cudaStream_t stream);
// two independent problems (same K, bf16-only epilogue) in one persistent launch
int gemm_bf16_dual(const GemmProblem& p1, const GemmProblem& p2, cudaStream_t stream);
// number of partial-logit slots a GATE epilogue writes for this problem
int gemm_gate_parts(const GemmProblem& p);

// Count + scatter (+ optional row gather) of (token, slot) pairs grouped by
// key = ids[p] / key_div, groups padded to row_tile rows (dice_ops.cu).
int permute_launch(const int32_t* ids, const uint8_t* active, int64_t n, int k, int groups,
                   int key_div, int row_tile, int experts_total, const uint16_t* rows, int hp,
                   uint16_t* x_perm, int32_t* pos, int32_t* tile_offsets, int64_t* counters,
                   int devices, int64_t row0, int64_t rows_total, int32_t* scratch,
                   cudaStream_t stream, int32_t* row_pair = nullptr);

}  // namespace dice
