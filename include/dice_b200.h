/*
 * dice_b200.h — C ABI of the B200-native DICE expert-parallel MoE sampling path.
 *
 * The reference (dicesim, /root/reference/pkg/src/dicesim) has no FFI: its
 * boundary is the set of module-level Python functions the schedule engine
 * imports (schedules.py:35-39, oracle.py:27-31). Each entry point below is the
 * device replacement for one of those functions; the Python package
 * paper_2411_16786_b200 binds them with ctypes and keeps the reference names
 * and signatures.
 *
 * Conventions
 *  - All pointers are caller-owned DEVICE pointers unless noted; no entry
 *    point allocates device memory or synchronises the host.
 *  - `stream` is a cudaStream_t passed as void*; every call is stream-ordered.
 *  - Feature dims are padded: hp = round_up(hidden_dim, 64), ep =
 *    round_up(expert_dim, 64); padded columns are zero and stay zero.
 *  - bf16 = IEEE bfloat16 bits (uint16), f32 = float, ids = int32.
 *  - Return 0 on success, else a DICE_ERR_* code that the Python layer maps
 *    1:1 onto the reference exception types (errors.py:4-29).
 *  - Non-finite values never return an error synchronously: kernels record
 *    the first offending step in a device `status` word (int32[4], see
 *    dice_status_reset) that the host reads once per run, raising
 *    NumericalDivergenceError(step) (schedules.py:445-449, 459-469).
 */
#ifndef DICE_B200_H_
#define DICE_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DICE_OK 0
#define DICE_ERR_CONTRACT 1   /* ContractError      (errors.py:12-13) */
#define DICE_ERR_CONFIG 2     /* ConfigurationError (errors.py:8-9)   */
#define DICE_ERR_NUMERICS 3   /* NumericsError      (errors.py:16-17) */
#define DICE_ERR_CUDA 4       /* CUDA launch / driver failure          */

/* Cond-comm strategies (policies.py:29-33). */
#define DICE_COND_OFF 0
#define DICE_COND_LOW_SCORE 1
#define DICE_COND_HIGH_SCORE 2
#define DICE_COND_RANDOM 3

/* GEMM epilogues of dice_gemm. */
#define DICE_EPI_STORE_BF16 0
#define DICE_EPI_GELU_BF16 1
#define DICE_EPI_STORE_F32 2
#define DICE_EPI_GELU_RESID 3

/* Library version / build identification (sm_100a). */
int dice_version(void);

/* CUDA events for stage timing that survive CUDA-graph capture (recorded as
 * external event nodes while the stream is capturing). */
int dice_event_create(void** event);
int dice_event_destroy(void* event);
int dice_event_record(void* event, void* stream);
int dice_event_elapsed_ms(void* start, void* end, float* ms);

/* status[0] = first step with a non-finite value (INT32_MAX if none),
 * status[1] = layer of the first non-finite gate input, status[2..3] reserved. */
int dice_status_reset(int32_t* status, void* stream);

/* splitmix64 stream -> uniform[-a, a) values, bit-exact in fp64.
 * Replaces splitmix64 + bits_to_uniform + init_model/sample_x0 consumption
 * order (model.py:28-36, 47-50, 133-162, 181-186). Element (r, c) of the
 * logical row-major [rows, cols] matrix is stream output start + r*cols + c.
 * transpose=0 writes out[r*ld + c]; transpose=1 writes out[c*ld + r].
 * out_dtype: 0 = f64, 1 = f32, 2 = bf16 (bf16 = RN(RN_f32(value))). */
int dice_splitmix_fill(uint64_t seed, uint64_t start, int64_t rows, int64_t cols,
                       double halfwidth, int transpose, int out_dtype, void* out,
                       int64_t ld, void* stream);

/* Raw splitmix64 outputs start..start+count-1 (model.py:28-36). */
int dice_splitmix_bits(uint64_t seed, uint64_t start, int64_t count, uint64_t* out,
                       void* stream);

/* Fused gate: logits = u[:, :h] @ w_gate, softmax over E, stable top-k on
 * scores (ties -> lower id), renormalised gates (model.py:209-223).
 * u: f32 [n, hp]; w_gate_t: f32 [E, hp] (transposed W_gate); ids: int32 [n, k];
 * gates: f32 [n, k]; scores: f32 [n, E] or NULL. Non-finite u records
 * (step, layer) into status (model.py:212-213). */
int dice_gate_topk(const float* u, const float* w_gate_t, int64_t n, int hp, int E, int k,
                   int32_t* ids, float* gates, float* scores, int32_t* status, int step,
                   int layer, void* stream);

/* dice_gate_topk followed, in the same kernel, by the conditional-communication
 * decision of each token on its fresh ids (dice_cond_decide's arguments and
 * semantics; the engine's gate + TokenCache.decide in one launch). */
int dice_gate_topk_decide(const float* u, const float* w_gate_t, int64_t n, int hp, int E, int k,
                          int32_t* ids, float* gates, float* scores, int32_t* status, int step,
                          int layer, int force, int refresh_interval, int strategy, int strict,
                          uint64_t random_key, int32_t* last_refresh, uint8_t* primed,
                          uint8_t* reduced, const int32_t* cached_ids, uint8_t* active,
                          uint8_t* write, void* stream);

/* Conditional-communication decision for one layer (TokenCache.decide,
 * policies.py:159-186 with reduced_slots 118-139, random_keep_slots 107-115).
 * State (this layer): last_refresh int32 [n] (init -1e9), primed uint8 [n],
 * reduced uint8 [n, k], cached_ids int32 [n, k] (read only when strict).
 * random_key = mix64(mix64(mix64(seed ^ TAG) + layer) + step), computed by
 * the caller (policies.py:113-114); token t's kept slot is
 * splitmix64(random_key, t+1) % k, so a shard whose first token is global row
 * row0 passes random_key + row0 * 0x9E3779B97F4A7C15 (mod 2^64).
 * Outputs active / write uint8 [n, k]. */
int dice_cond_decide(const int32_t* ids, int64_t n, int k, int step, int force,
                     int refresh_interval, int strategy, int strict, uint64_t random_key,
                     int32_t* last_refresh, uint8_t* primed, uint8_t* reduced,
                     const int32_t* cached_ids, uint8_t* active, uint8_t* write,
                     void* stream);

/* Token permute (block prefix-sum) for routed_rows' (slot, expert) grouping
 * (model.py:255-276) and the all-to-all byte plan (cluster.py:82-109).
 * Pairs (t, s) with active[t, s] (active NULL = all) are assigned rows of the
 * expert-sorted, 256-row-padded buffer: pos[t, s] = row or -1. Within an
 * expert, rows follow token-major pair order (deterministic; GEMM rows are
 * independent so the reference's slot-major grouping changes no value).
 * tile_offsets: int32 [E+1] 256-row m-tile prefix per expert (device-resident; feeds
 * the grouped GEMM with no host sync). counters: int64 [2] accumulated
 * {active pairs, active pairs whose expert lives off the token's home device}
 * under placement expert_dev = e / (E/D), home = ((row0+t)*D)/R_total.
 * Also gathers x_perm[pos] = u16[t] (bf16 [max_rows, hp]). */
int dice_route_permute(const int32_t* ids, const uint8_t* active, int64_t n, int k, int E,
                       const uint16_t* u16, int hp, uint16_t* x_perm, int64_t max_rows,
                       int32_t* pos, int32_t* tile_offsets, int64_t* counters,
                       int devices, int64_t row0, int64_t rows_total, int32_t* scratch,
                       int32_t* row_pair, void* stream);

/* Router + conditional-communication decision + token permute in ONE launch
 * (single-GPU engine, E = 8 or 16, k <= E): dice_gate_topk(_decide) (decide = 0 / 1)
 * whose blocks of 256/E tokens also group their active pairs by expert and copy
 * the tokens' rows, rounded to bf16 from the fp32 u (the bits the local GEMM
 * stores as its bf16 output), to their permuted rows. Expert e owns rows
 * [e*cap, (e+1)*cap) of x_perm (bf16 [E*cap, hp], cap >= n, a multiple of
 * 256); a block's rows of expert e follow pair order t*k+s and start at the
 * offset one atomic add on the expert's row counter returned, so the order of
 * the blocks within a region varies between launches (no value does: every
 * expert-FFN output row depends on its own row only). Outputs pos int32 [n, k]
 * (-1 inactive), row_pair int32 [E*cap] (pair of each row, -1 on the padding
 * rows up to each expert's 256-row tile end), tile_offsets int32 [E+1] (256-row
 * tile prefix, for dice_expert_gemm1_with_dense(group_stride = cap)) and adds
 * dice_route_permute's counters. route_state: uint64
 * [dice_gate_route_state_words(n)], zero-filled once, then owned by these
 * launches (a finished-block ticket and the per-expert row counters, reset by
 * the last block of every launch). */
int64_t dice_gate_route_state_words(int64_t n);
int dice_gate_route(const float* u, const float* w_gate_t, int64_t n, int hp, int E, int k,
                    int32_t* ids, float* gates, float* scores, int32_t* status, int step,
                    int layer, int decide, int force, int refresh_interval, int strategy,
                    int strict, uint64_t random_key, int32_t* last_refresh, uint8_t* primed,
                    uint8_t* reduced, const int32_t* cached_ids, uint8_t* active,
                    uint8_t* write, uint16_t* x_perm, int64_t cap, int32_t* pos,
                    int32_t* row_pair, int32_t* tile_offsets, int64_t* counters, int devices,
                    int64_t rows_total, uint64_t* route_state, void* stream);

/* Upper bound of rows of the padded permuted buffer for n*k pairs over E experts. */
int64_t dice_permute_max_rows(int64_t n, int k, int E);

/* int32 words of scratch dice_route_permute needs (per-block expert counts). */
int64_t dice_permute_scratch_ints(int64_t n, int k, int E);

/* Grouped expert FFN on the permuted rows (expert_forward, model.py:226-232):
 * hbuf = gelu(x_perm @ W1_e) (bf16 [max_rows, ep]); y = hbuf @ W2_e (bf16 [max_rows, hp]).
 * w1_t: bf16 [E*ep, hp] (per expert W1^T); w2_t: bf16 [E*hp, ep] (per expert W2^T).
 * tcgen05/TMEM/TMA grouped GEMM, tile -> expert from tile_offsets. */
int dice_grouped_ffn(const uint16_t* x_perm, int64_t max_rows, const uint16_t* w1_t,
                     const uint16_t* w2_t, int E, int hp, int ep, const int32_t* tile_offsets,
                     uint16_t* hbuf, uint16_t* y, void* stream);

/* Stale-activation cache merge + weighted routed sum (TokenCache.assemble,
 * policies.py:188-208; combine_outputs' routed part, model.py:295-298) — the
 * functional API form (policies.TokenCache.assemble, model.routed_rows).
 * For each token t: routed[t] = sum_s g_s * row_s (slots left to right, f32)
 * where active pairs take row y[pos[t,s]] and gate gates[t,s], inactive pairs
 * take the cached row/gate. Pairs with write[t,s] store their fresh row/gate/id
 * into the cache. cache_* may be NULL (cond-comm off). rows_out (f32 [k, n, hp])
 * and gates_out (f32 [n, k]) are optional. */
int dice_cache_assemble(const uint16_t* y, const int32_t* pos, const uint8_t* active,
                        const uint8_t* write, const float* gates, const int32_t* ids,
                        int64_t n, int k, int hp, uint16_t* cache_rows, float* cache_gates,
                        int32_t* cache_ids, float* routed, float* rows_out, float* gates_out,
                        void* stream);

/* Dense bf16 GEMM C[M, N] = A[M, K] @ B[N, K]^T with a fused epilogue (see
 * DICE_EPI_*): local_block (model.py:244-252) = GELU_RESID with residual h;
 * shared_forward GEMM1 (model.py:235-241) = GELU_BF16 with the S experts
 * concatenated on N, GEMM2 = STORE_F32. */
int dice_gemm(int epi, const uint16_t* A, int64_t M, const uint16_t* B, int N, int K,
              float* out_f32, int64_t ld_f32, uint16_t* out_bf16, int64_t ld_bf16,
              const float* residual, int64_t ld_res, void* stream);

/* The two halves of dice_grouped_ffn, the first merged with a dense GELU GEMM
 * of the same K in ONE persistent launch: hbuf = gelu(x_perm W1_e) over the
 * expert tiles AND out2 [M2, N2] = gelu(A2 B2^T) (the stage's shared-expert
 * GEMM1, shared_forward model.py:235-241, A2 = u bf16 [M2, hp], B2 = ws1_t);
 * then y = hbuf W2_e (expert_forward model.py:226-232). group_stride = 0:
 * x_perm holds the experts' 256-row tiles contiguously (dice_route_permute,
 * max_rows rows); > 0: expert e's rows start at row e * group_stride
 * (dice_gate_route's capacity regions, E * group_stride rows). hbuf is
 * tile-contiguous either way (max_rows rows). */
int dice_expert_gemm1_with_dense(const uint16_t* x_perm, int64_t max_rows, int64_t group_stride,
                                 const uint16_t* w1_t, int E, int hp, int ep,
                                 const int32_t* tile_offsets, uint16_t* hbuf, const uint16_t* A2,
                                 int64_t M2, const uint16_t* B2, int N2, uint16_t* out2,
                                 void* stream);
int dice_expert_gemm2(const uint16_t* hbuf, int64_t max_rows, const uint16_t* w2_t, int E, int hp,
                      int ep, const int32_t* tile_offsets, uint16_t* y, void* stream);

/* The engine's routed combine, split between the producer and the consumer of
 * a layer's expert rows (TokenCache.assemble policies.py:188-208 +
 * combine_outputs model.py:279-298 + _consume schedules.py:308-317), with no
 * kernel in between:
 *
 * dice_expert_gemm2_pairs: the expert GEMM2 (y = hbuf W2_e per expert tile)
 * whose epilogue stores the bf16 row of permuted row r (pair p = row_pair[r] =
 * t*k + s from dice_route_permute / dice_gate_route, -1 on padding; with
 * pair_group_stride > 0 the map is indexed in dice_gate_route's capacity
 * regions: tile j of expert e -> rows e * stride + 256 j ...) into pair_rows[s][t]
 * ([k, n, hp]: the layer's token-cache rows) and persists gates[p] / ids[p]
 * into cache_gates[p] / cache_ids[p] (either may be NULL). Every computed
 * pair is persisted: a cached entry is only ever read for a reduced pair that
 * is not due, and a pair enters the reduced set only at a refresh, which
 * writes it (policies.py:171-186), so persisting the other fresh pairs too
 * leaves every value the reference reads unchanged — the rows / gates then
 * hold, per pair, its latest computed row and gate: for an active pair the
 * fresh one, for an inactive pair the cached one (policies.py:197-202).
 *
 * dice_gemm_consume: out = residual + ((A B^T + g_0 row_0) + g_1 row_1 ...)
 * with row_s = pair_rows[s][t], g_s = pair_gates[t][s] — the shared-expert
 * GEMM2 with the layer's consume in its epilogue (slots left to right, the
 * product and each sum rounded; then the residual, schedules.py:317) ->
 * out_f32 / out_bf16. dice_consume_rows: the same without shared experts
 * (S = 0): out = residual + ((0 + g_0 row_0) + ...). */
int dice_expert_gemm2_pairs(const uint16_t* hbuf, int64_t max_rows, const uint16_t* w2_t, int E,
                            int hp, int ep, const int32_t* tile_offsets, const int32_t* row_pair,
                            int64_t pair_group_stride, const float* gates, const int32_t* ids,
                            int k, int64_t n, uint16_t* pair_rows, float* cache_gates,
                            int32_t* cache_ids, void* stream);
int dice_gemm_consume(const uint16_t* A, int64_t M, const uint16_t* B, int N, int K,
                      const float* residual, int64_t ld_res, const uint16_t* pair_rows,
                      const float* pair_gates, int k, float* out_f32, int64_t ld_f32,
                      uint16_t* out_bf16, int64_t ld_bf16, void* stream);
int dice_consume_rows(const float* residual, const uint16_t* pair_rows, const float* pair_gates,
                      int64_t n, int k, int hp, float* out, uint16_t* out_bf16, void* stream);

/* out[t] = base[t] + sum_s gates[t, s] * rows[s, t] (f32, combine_outputs
 * model.py:279-298 and the consume residual, schedules.py:317). rows f32
 * [k, n, hp]; base f32 [n, hp]; optional residual adds u first:
 * out = residual + (base + sum). */
int dice_combine(const float* base, const float* rows, const float* gates, const float* residual,
                 int64_t n, int k, int hp, float* out, uint16_t* out_bf16, void* stream);

/* x_{s+1} = x_s - eta * y (model.py:301-305), f32 in place, plus its bf16 copy;
 * records `step` into status on a non-finite result (schedules.py:447-449). */
int dice_denoise(float* x, uint16_t* x16, const float* y, float eta, int64_t n, int hp,
                 int32_t* status, int step, void* stream);

/* Adjacent-step drift of one layer (step_similarity / _cosine, model.py:308-346):
 * out f64 [4] = {sum a*b, sum a*a, sum b*b over the first `cols` columns of the
 * n rows of a = prev (ld_prev) and b = cur (ld_cur), number of rows t with
 * prev_top[t * top_stride] == cur_ids[t * k]} (top-1 routing agreement).
 * Deterministic fixed-order fp64 reductions. roll != 0 then stores cur into
 * prev and cur's top-1 into prev_top (a runner's previous-step buffers).
 * partials: f64 [dice_similarity_partial_words()] scratch. */
int64_t dice_similarity_partial_words(void);
int dice_step_similarity(float* prev, const float* cur, int64_t n, int cols, int64_t ld_prev,
                         int64_t ld_cur, int32_t* prev_top, int64_t top_stride,
                         const int32_t* cur_ids, int k, int roll, double* partials, double* out,
                         void* stream);

/* f32 [n, ld_in] (first `cols` columns) -> bf16 [n, hp] and f32 [n, hp] padded copies. */
int dice_pack_rows(const float* in, int64_t n, int cols, int64_t ld_in, int hp, float* out32,
                   uint16_t* out16, void* stream);

/* ------------------------------------------------------------------------
 * Expert parallelism over peer memory (one process per GPU, NVLink/NVSwitch).
 * Replaces the simulated dispatch / combine all-to-alls (schedules.py:326,
 * 332, 376, 393; cluster.py:93-109) with P2P stores into IPC-shared windows.
 * ------------------------------------------------------------------------ */

/* cudaMalloc + zero fill (windows must be whole allocations to be IPC-shared). */
int dice_device_alloc(int64_t bytes, void** ptr);
int dice_device_free(void* ptr);

/* CUDA IPC: 64-byte handle of a dice_device_alloc allocation; open / close a
 * peer's handle (not the caller's own). */
int dice_ipc_get_handle(const void* dev_ptr, uint8_t* handle64);
int dice_ipc_open(const uint8_t* handle64, void** dev_ptr);
int dice_ipc_close(void* dev_ptr);

/* Batched stream memory operations on 32-bit flags (addrs: host array of
 * device addresses, local or peer-mapped). wait: the stream stalls until every
 * flag == value. write: each write is ordered after (and fenced against) prior
 * work on the stream. Both are captured by CUDA graphs. */
int dice_stream_wait_eq(const uint64_t* addrs, int count, uint32_t value, void* stream);
int dice_stream_write(const uint64_t* addrs, int count, uint32_t value, void* stream);

/* Dispatch all-to-all send of one layer: groups this rank's active pairs by
 * destination rank (expert e lives on rank e/(E/D)), accumulates
 * {active pairs, remote pairs} in counters, and stores each pair's bf16 row
 * and int4 metadata {local expert, home pair index t*k+s, gate (f32 bits),
 * expert id} into the destination's window region for source `me`, plus the
 * per-destination row count. rx_*: host arrays of D device pointers to those
 * regions. gates f32 [n, k]; pos_dest int32 [n*k], dest_offsets int32 [D+1],
 * scratch >= dice_permute_scratch_ints(n, k, D). */
int dice_ep_dispatch(const int32_t* ids, const float* gates, const uint8_t* active, int64_t n,
                     int k, int E, int D, int me, const uint16_t* u16, int hp, int32_t* pos_dest,
                     int32_t* dest_offsets, int64_t* counters, int64_t row0, int64_t rows_total,
                     int32_t* scratch, const uint64_t* rx_rows, const uint64_t* rx_meta,
                     const uint64_t* rx_count, void* stream);

/* Expert side of one layer: groups the D*cap window rows by local expert,
 * runs the grouped expert FFN (expert_forward, model.py:226-232); the expert
 * GEMM2's epilogue stores every finished row straight into its home rank's
 * pair rows [k, n_home, hp] at [s][t] with its gate and expert id (the combine
 * all-to-all fused into the GEMM, as peer-memory stores; the persistence rule
 * of dice_expert_gemm2_pairs). home_rows / home_gates / home_ids: host arrays
 * of D device pointers (the layer's pair rows / cache gates / cache ids of
 * every rank, peer-mapped), home_n: host array of the D ranks' row counts.
 * A2 != NULL: the rank's dense shared-expert GEMM1 out2 = gelu(A2 B2^T)
 * [M2, N2] runs in the same GEMM1 launch. row_pair: int32 [max_rows]. */
int dice_ep_expert(const uint16_t* rx_rows, const void* rx_meta, const int32_t* rx_count, int D,
                   int64_t cap, int El, int hp, int ep, int k, const uint16_t* w1_t,
                   const uint16_t* w2_t, int32_t* ids_rx, int32_t* pos_rx, int32_t* tile_offsets,
                   int32_t* scratch, uint16_t* x_perm, int64_t max_rows, uint16_t* hbuf,
                   int32_t* row_pair, const uint64_t* home_rows, const uint64_t* home_gates,
                   const uint64_t* home_ids, const int64_t* home_n, const uint16_t* A2,
                   int64_t M2, const uint16_t* B2, int N2, uint16_t* out2, void* stream);

/* dice_ep_expert in two parts, so the exchange's receive-side regroup (a
 * communication cost) is timed apart from the expert FFN:
 * dice_ep_regroup: window rows -> x_perm grouped by local expert (256-row
 * tiles, tile_offsets, row_pair = window entry of each row, -1 on padding);
 * dice_ep_expert_ffn: grouped FFN on x_perm whose GEMM2 epilogue stores into
 * the home ranks' pair rows (arguments as dice_ep_expert). */
int dice_ep_regroup(const uint16_t* rx_rows, const void* rx_meta, const int32_t* rx_count, int D,
                    int64_t cap, int El, int hp, int32_t* ids_rx, int32_t* pos_rx,
                    int32_t* tile_offsets, int32_t* scratch, uint16_t* x_perm, int32_t* row_pair,
                    void* stream);
int dice_ep_expert_ffn(const uint16_t* x_perm, int64_t max_rows, const void* rx_meta,
                       int64_t cap, int D, int El, int hp, int ep, int k, const uint16_t* w1_t,
                       const uint16_t* w2_t, const int32_t* tile_offsets, uint16_t* hbuf,
                       const int32_t* row_pair, const uint64_t* home_rows,
                       const uint64_t* home_gates, const uint64_t* home_ids,
                       const int64_t* home_n, const uint16_t* A2, int64_t M2, const uint16_t* B2,
                       int N2, uint16_t* out2, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DICE_B200_H_ */
