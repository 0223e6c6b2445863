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
  // consume (schedules.py:308-317, model.py:279-298): the shared-expert GEMM2
  // accumulator plus the token's routed rows, slots left to right, then the
  // residual: v = residual + ((acc + g_0 * row_0) + g_1 * row_1 ...) with
  // row_s = pair_rows[s][t] (bf16 [k, n, N]) and g_s = pair_gates[t][s]
  // (f32 [n, k]) -> out_f32, out_bf16
  EPI_CONSUME = 4,
  // single-GPU expert GEMM2: the finished row of permuted row r (pair p =
  // row_pair[r] = t*k + s; -1 on padding rows) is stored as bf16 at
  // out_bf16[s][t] ([k, n, N]: the layer's pair rows, i.e. the token cache
  // rows), and its gate / expert id at cache_gates[p] / cache_ids[p]
  EPI_STORE_PAIR = 5,
  // expert-parallel expert GEMM2 with the combine all-to-all fused: the row of
  // window entry i = row_pair[r] (source rank i / scatter_cap, metadata int4
  // {local expert, home pair, gate bits, global expert}) is stored as bf16
  // straight into that rank's pair rows (peer memory) at [s][t] of its home
  // pair, with the gate and expert id, tile by tile as the GEMM finishes them
  EPI_STORE_SCATTER = 6,
};

constexpr int kMaxRanks = 16;

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
  int stages;            // operand ring depth actually used (set by the host)
  // grouped GEMMs over capacity-strided expert regions (the fused router
  // writes expert e's permuted rows at e * stride): A rows of group g's tile j
  // start at g * a_group_stride + 256 j (0: tiles are contiguous, row 256 m);
  // STORE_PAIR's row -> pair map is indexed the same way with pair_group_stride
  int64_t a_group_stride;
  int64_t pair_group_stride;
  // CONSUME: pair_rows bf16 [k, n_tokens, ld_bf16-wide rows], pair_gates f32 [n, k]
  // STORE_PAIR: row -> pair map, source gates / ids of the pairs [n, k], the
  // cache gates / ids they are persisted to
  const __nv_bfloat16* pair_rows;
  const int32_t* row_pair;
  const float* pair_gates;
  const int32_t* pair_ids;
  float* cache_gates;
  int32_t* cache_ids;
  int top_k;
  int64_t n_tokens;
  // STORE_SCATTER: window metadata int4 [D * cap], entries per source rank, and
  // per source rank the (peer-mapped) pair rows / gates / ids of the layer and
  // its row count
  const void* scatter_meta;
  int64_t scatter_cap;
  uint64_t scatter_rows[kMaxRanks];
  uint64_t scatter_gates[kMaxRanks];
  uint64_t scatter_ids[kMaxRanks];
  int64_t scatter_n[kMaxRanks];
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

// Count + scatter (+ optional row gather) of (token, slot) pairs grouped by
// key = ids[p] / key_div, groups padded to row_tile rows (dice_ops.cu).
int permute_launch(const int32_t* ids, const uint8_t* active, int64_t n, int k, int groups,
                   int key_div, int row_tile, int experts_total, const uint16_t* rows, int hp,
                   uint16_t* x_perm, int32_t* pos, int32_t* tile_offsets, int64_t* counters,
                   int devices, int64_t row0, int64_t rows_total, int32_t* scratch,
                   cudaStream_t stream, int32_t* row_pair = nullptr);

}  // namespace dice
