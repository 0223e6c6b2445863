// Expert-parallel token exchange over peer memory (NVLink / NVSwitch).
//
// One process per GPU. Every rank exports its receive windows with CUDA IPC;
// peers map them and the send kernels store token rows straight into the
// owner's window (the permute writes the all-to-all), so there is no staging
// copy and no host synchronisation. Completion is signalled with constant
// valued ready/free flags driven by batched stream memory operations
// (cuStreamBatchMemOp wait/write), which CUDA graphs capture, so a whole
// sampling run replays as one graph on every rank.
//
// Reference semantics: the dispatch all-to-all moves the active (token, slot)
// pairs to the rank owning the expert (schedules.py:326, cluster.py:93-109);
// the combine all-to-all returns the expert rows to the token's home rank
// (schedules.py:332, 393); expert e lives on rank e / (E/D) and token t on
// rank (t*D)/R (cluster.py:61-72).
#include <cstring>
#include <mutex>

#include "dice_gemm.h"
#include "dice_ptx.cuh"

namespace dice {

struct PeerPtrs {
  void* p[kMaxRanks];
};

// Sender: warp per active pair; rows go to the destination rank's window at
// the pair's compact index within (me -> dest), metadata {local expert, home
// pair, gate bits, expert id}.
__global__ void __launch_bounds__(256) ep_send_kernel(
    const int32_t* __restrict__ ids, const float* __restrict__ gates,
    const int32_t* __restrict__ pos_dest, const int32_t* __restrict__ dest_offsets,
    int64_t pairs, int k, int El, const uint16_t* __restrict__ u16, int hp, PeerPtrs rx_rows,
    PeerPtrs rx_meta, PeerPtrs rx_count, int D) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  if (blockIdx.x == 0 && threadIdx.x < D) {
    const int d = threadIdx.x;
    *reinterpret_cast<int32_t*>(rx_count.p[d]) = dest_offsets[d + 1] - dest_offsets[d];
  }
  const int vec = hp / 8;
  for (int64_t q = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; q < pairs;
       q += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int pd = pos_dest[q];
    if (pd < 0) continue;
    const int e = ids[q];
    const int d = e / El;
    const int idx = pd - dest_offsets[d];
    const uint4* src = reinterpret_cast<const uint4*>(u16 + (q / k) * hp);
    uint4* dst = reinterpret_cast<uint4*>(static_cast<uint16_t*>(rx_rows.p[d]) + (int64_t)idx * hp);
    for (int c = lane; c < vec; c += 32) dst[c] = src[c];
    if (lane == 0)
      static_cast<int4*>(rx_meta.p[d])[idx] = make_int4(e - d * El, (int)q, __float_as_int(gates[q]), e);
  }
}

// Receiver: expert key of every received row (-1 beyond each source's count).
__global__ void ep_rx_ids_kernel(const int4* __restrict__ meta, const int32_t* __restrict__ counts,
                                 int D, int64_t cap, int32_t* ids_rx) {
  pdl_enter();
  const int64_t total = (int64_t)D * cap;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int src = (int)(g / cap);
    const int64_t j = g - (int64_t)src * cap;
    ids_rx[g] = j < counts[src] ? meta[g].x : -1;
  }
}

namespace {

typedef CUresult (*BatchMemOpFn)(CUstream, unsigned int, CUstreamBatchMemOpParams*, unsigned int);

BatchMemOpFn batch_memop() {
  static BatchMemOpFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamBatchMemOp", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<BatchMemOpFn>(p);
  });
  return fn;
}

PeerPtrs table(const uint64_t* ptrs, int D, int64_t offset_bytes) {
  PeerPtrs t;
  memset(&t, 0, sizeof(t));
  for (int d = 0; d < D; ++d)
    t.p[d] = reinterpret_cast<void*>(ptrs[d] + (uint64_t)offset_bytes);
  return t;
}

int grid_warps(int64_t warps) {
  int64_t g = (warps * 32 + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  return g < 1 ? 1 : (int)g;
}

}  // namespace
}  // namespace dice

using namespace dice;

extern "C" {

int dice_device_alloc(int64_t bytes, void** ptr) {
  if (bytes <= 0) return DICE_ERR_CONTRACT;
  if (cudaMalloc(ptr, (size_t)bytes) != cudaSuccess) return DICE_ERR_CUDA;
  return cudaMemset(*ptr, 0, (size_t)bytes) == cudaSuccess ? DICE_OK : DICE_ERR_CUDA;
}

int dice_device_free(void* ptr) { return cudaFree(ptr) == cudaSuccess ? DICE_OK : DICE_ERR_CUDA; }

int dice_ipc_get_handle(const void* dev_ptr, uint8_t* handle64) {
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)) != cudaSuccess) return DICE_ERR_CUDA;
  memcpy(handle64, &h, sizeof(h));
  return DICE_OK;
}

int dice_ipc_open(const uint8_t* handle64, void** dev_ptr) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  return cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess
             ? DICE_OK : DICE_ERR_CUDA;
}

int dice_ipc_close(void* dev_ptr) {
  return cudaIpcCloseMemHandle(dev_ptr) == cudaSuccess ? DICE_OK : DICE_ERR_CUDA;
}

// Stream-ordered waits until every 32-bit flag at addrs[i] equals `value`
// (one batched memop; the stream stalls on the device, no SM spins).
int dice_stream_wait_eq(const uint64_t* addrs, int count, uint32_t value, void* stream) {
  BatchMemOpFn fn = batch_memop();
  if (fn == nullptr || count < 0 || count > 64) return DICE_ERR_CUDA;
  if (count == 0) return DICE_OK;
  // the ready flags are written by peer GPUs after their P2P row stores: where
  // the device supports it, the wait also flushes outstanding remote writes so
  // the rows are visible to the kernels behind it
  static const unsigned flush = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&v, cudaDevAttrCanFlushRemoteWrites, dev) != cudaSuccess) {
      cudaGetLastError();
      v = 0;
    }
    return v ? (unsigned)CU_STREAM_WAIT_VALUE_FLUSH : 0u;
  }();
  CUstreamBatchMemOpParams ops[64];
  memset(ops, 0, sizeof(ops));
  for (int i = 0; i < count; ++i) {
    ops[i].waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_32;
    ops[i].waitValue.address = (CUdeviceptr)addrs[i];
    ops[i].waitValue.value = value;
    ops[i].waitValue.flags = CU_STREAM_WAIT_VALUE_EQ | flush;
  }
  return fn((CUstream)stream, (unsigned)count, ops, 0) == CUDA_SUCCESS ? DICE_OK : DICE_ERR_CUDA;
}

// Stream-ordered 32-bit writes (each preceded by a fence over prior stream work).
int dice_stream_write(const uint64_t* addrs, int count, uint32_t value, void* stream) {
  BatchMemOpFn fn = batch_memop();
  if (fn == nullptr || count < 0 || count > 64) return DICE_ERR_CUDA;
  if (count == 0) return DICE_OK;
  CUstreamBatchMemOpParams ops[64];
  memset(ops, 0, sizeof(ops));
  for (int i = 0; i < count; ++i) {
    ops[i].writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_32;
    ops[i].writeValue.address = (CUdeviceptr)addrs[i];
    ops[i].writeValue.value = value;
    ops[i].writeValue.flags = CU_STREAM_WRITE_VALUE_DEFAULT;
  }
  return fn((CUstream)stream, (unsigned)count, ops, 0) == CUDA_SUCCESS ? DICE_OK : DICE_ERR_CUDA;
}

// Dispatch send for one layer (TokenCache.decide has produced `active`).
// Groups this rank's active pairs by destination rank (compact, no padding),
// counts bytes of remote pairs, and stores every row + {local expert, pair,
// gate, expert} into the destination's window region reserved for this source
// rank. rx_rows/rx_meta/rx_count: per-destination device pointers (peer-mapped)
// to this layer's region for source `me`.
int dice_ep_dispatch(const int32_t* ids, const float* gates, const uint8_t* active, int64_t n,
                     int k, int E, int D, int me, const uint16_t* u16, int hp, int32_t* pos_dest,
                     int32_t* dest_offsets, int64_t* counters, int64_t row0, int64_t rows_total,
                     int32_t* scratch, const uint64_t* rx_rows, const uint64_t* rx_meta,
                     const uint64_t* rx_count, void* stream) {
  if (D < 1 || D > kMaxRanks || E % D != 0 || hp % 64 != 0 || me < 0 || me >= D ||
      gates == nullptr)
    return DICE_ERR_CONTRACT;
  cudaStream_t s = (cudaStream_t)stream;
  const int El = E / D;
  int rc = permute_launch(ids, active, n, k, D, El, 1, E, nullptr, hp, nullptr, pos_dest,
                          dest_offsets, counters, D, row0, rows_total, scratch, s);
  if (rc) return rc;
  // plain launches on the exchange path: these kernels follow stream memory
  // operations (flag waits), not kernels
  ep_send_kernel<<<grid_warps(n * k), 256, 0, s>>>(ids, gates, pos_dest, dest_offsets, n * k, k,
                                                   El, u16, hp, table(rx_rows, D, 0),
                                                   table(rx_meta, D, 0), table(rx_count, D, 0), D);
  return cudaGetLastError() == cudaSuccess ? DICE_OK : DICE_ERR_CUDA;
}

// Receive side of one layer, part 1 (the exchange's regroup): group the rows
// every source rank stored in this rank's window by local expert (256-row
// padded tiles of x_perm, row_pair = window entry of each row, -1 on padding).
// rx_rows [D*cap, hp], rx_meta [D*cap] (int4), rx_count [D] are this rank's
// window for the layer.
int dice_ep_regroup(const uint16_t* rx_rows, const void* rx_meta, const int32_t* rx_count, int D,
                    int64_t cap, int El, int hp, int32_t* ids_rx, int32_t* pos_rx,
                    int32_t* tile_offsets, int32_t* scratch, uint16_t* x_perm, int32_t* row_pair,
                    void* stream) {
  if (D < 1 || D > kMaxRanks || hp % 64 != 0 || El < 1 || row_pair == nullptr)
    return DICE_ERR_CONTRACT;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t total = (int64_t)D * cap;
  ep_rx_ids_kernel<<<(int)((total + 255) / 256 < 2368 ? (total + 255) / 256 : 2368), 256, 0, s>>>(
      static_cast<const int4*>(rx_meta), rx_count, D, cap, ids_rx);
  return permute_launch(ids_rx, nullptr, total, 1, El, 1, 256, El, rx_rows, hp, x_perm, pos_rx,
                        tile_offsets, nullptr, 1, 0, total, scratch, s, row_pair);
}

// Part 2: the grouped expert FFN on the regrouped rows; GEMM1 (+ the rank's
// shared GEMM1 in the same launch when A2 != NULL), then GEMM2 whose
// epilogue stores every finished row into its home rank's pair rows (with
// gate and expert id from the window metadata) over peer memory.
int dice_ep_expert_ffn(const uint16_t* x_perm, int64_t max_rows, const void* rx_meta,
                       int64_t cap, int D, int El, int hp, int ep, int k, const uint16_t* w1_t,
                       const uint16_t* w2_t, const int32_t* tile_offsets, uint16_t* hbuf,
                       const int32_t* row_pair, const uint64_t* home_rows,
                       const uint64_t* home_gates, const uint64_t* home_ids,
                       const int64_t* home_n, const uint16_t* A2, int64_t M2, const uint16_t* B2,
                       int N2, uint16_t* out2, void* stream) {
  if (D < 1 || D > kMaxRanks || hp % 64 != 0 || ep % 64 != 0 || El < 1 || k < 1 ||
      row_pair == nullptr)
    return DICE_ERR_CONTRACT;
  cudaStream_t s = (cudaStream_t)stream;
  int rc = dice_expert_gemm1_with_dense(x_perm, max_rows, 0, w1_t, El, hp, ep, tile_offsets, hbuf,
                                        A2, A2 != nullptr ? M2 : 0, B2, N2, out2, stream);
  if (rc) return rc;
  GemmProblem q{};
  q.A = hbuf; q.A_rows = max_rows; q.B = w2_t; q.M = (int)max_rows; q.N = hp; q.K = ep;
  q.num_groups = El; q.group_tile_offsets = tile_offsets; q.max_m_tiles = (int)(max_rows / 256);
  q.epi_kind = EPI_STORE_SCATTER;
  q.epi.ld_bf16 = hp;
  q.epi.row_pair = const_cast<int32_t*>(row_pair);
  q.epi.top_k = k;
  q.epi.scatter_meta = rx_meta;
  q.epi.scatter_cap = cap;
  for (int r = 0; r < D; ++r) {
    q.epi.scatter_rows[r] = home_rows[r];
    q.epi.scatter_gates[r] = home_gates[r];
    q.epi.scatter_ids[r] = home_ids[r];
    q.epi.scatter_n[r] = home_n[r];
  }
  return gemm_bf16(q, s);
}

// Both parts (regroup, then the FFN with the fused combine stores).
int dice_ep_expert(const uint16_t* rx_rows, const void* rx_meta, const int32_t* rx_count, int D,
                   int64_t cap, int El, int hp, int ep, int k, const uint16_t* w1_t,
                   const uint16_t* w2_t, int32_t* ids_rx, int32_t* pos_rx, int32_t* tile_offsets,
                   int32_t* scratch, uint16_t* x_perm, int64_t max_rows, uint16_t* hbuf,
                   int32_t* row_pair, const uint64_t* home_rows, const uint64_t* home_gates,
                   const uint64_t* home_ids, const int64_t* home_n, const uint16_t* A2,
                   int64_t M2, const uint16_t* B2, int N2, uint16_t* out2, void* stream) {
  if (ep % 64 != 0 || k < 1) return DICE_ERR_CONTRACT;
  int rc = dice_ep_regroup(rx_rows, rx_meta, rx_count, D, cap, El, hp, ids_rx, pos_rx,
                           tile_offsets, scratch, x_perm, row_pair, stream);
  if (rc) return rc;
  return dice_ep_expert_ffn(x_perm, max_rows, rx_meta, cap, D, El, hp, ep, k, w1_t, w2_t,
                            tile_offsets, hbuf, row_pair, home_rows, home_gates, home_ids, home_n,
                            A2, M2, B2, N2, out2, stream);
}

}  // extern "C"
