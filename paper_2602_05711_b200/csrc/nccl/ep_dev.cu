// Fused expert-parallel exchange on the NCCL 2.28 device API (include/omnimoe_ep.h; SURVEY
// §8(f) N3).  Built into libomnimoe_ep.so (links libnccl); the product library
// libomnimoe.so does not depend on it.
//
// Windows (symmetric, ncclMemAlloc + ncclCommWindowRegister): counts [R][R][2] int64, x_recv
// [row_cap][d] bf16, rec [rec_cap][3] int32, y_ret [row_cap][d] bf16.  With C[src][dst] =
// (rows, records) src sends dst:
//   * source src's block lands in dst's x_recv at row  sum_{s < src} C[s][dst].rows  and in
//     dst's rec at record  sum_{s < src} C[s][dst].records  (sources in rank order, the
//     layout the host-API path's all_to_all produces);
//   * the record slot (row within the source's block, omnimoe_ep_pack) becomes the
//     receiver's row index, so the receiver unpacks with one "source";
//   * dst returns its received row j (of source src, slot q) into src's y_ret at row
//     sum_{t < dst} C[src][t].rows + q  -- src's x_send position of that row.
// Ordering: kernel 1 stores this rank's counts row into every peer's counts window and
// crosses an LSA barrier (release / acquire: afterwards every rank's window holds the whole
// matrix); the copy kernels store into peers with plain vector stores; a barrier kernel after
// each copy makes the peers' stores visible before anyone reads its windows.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>

#include <cstdint>
#include <cstring>
#include <string>

#include "../../../include/omnimoe_ep.h"

struct omnimoe_ep_comm {
  ncclComm_t comm = nullptr;
  ncclDevComm dev{};
  int rank = 0, world = 1;
  int64_t d = 0, row_cap = 0, rec_cap = 0;
  void *counts = nullptr, *x = nullptr, *rec = nullptr, *y = nullptr;
  ncclWindow_t wc = nullptr, wx = nullptr, wr = nullptr, wy = nullptr;
};

namespace {
thread_local std::string g_err;
constexpr int kMaxR = 16;

omnimoe_status fail(const std::string& m, omnimoe_status s) {
  g_err = m;
  return s;
}
#define EP_NCCL(call)                                                                               \
  do {                                                                                            \
    ncclResult_t r__ = (call);                                                                    \
    if (r__ != ncclSuccess) return fail(std::string(#call) + ": " + ncclGetErrorString(r__), OMNIMOE_ERR_CUDA); \
  } while (0)
#define EP_LAUNCH(what)                                                                           \
  do {                                                                                            \
    cudaError_t e__ = cudaGetLastError();                                                         \
    if (e__ != cudaSuccess) return fail(std::string(what) + ": " + cudaGetErrorString(e__), OMNIMOE_ERR_CUDA); \
  } while (0)

// C[src][dst][k] in a counts window
__device__ __forceinline__ int64_t cnt(const int64_t* c, int R, int src, int dst, int k) {
  return c[((int64_t)src * R + dst) * 2 + k];
}

__device__ __forceinline__ void lsa_barrier(const ncclDevComm& dc) {
  ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamLsa(dc), dc.lsaBarrier, 0);
  bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
}

// kernel 1 (one CTA): this rank's counts row -> every peer's counts window, then a barrier
__global__ void ep_counts_kernel(ncclDevComm dc, ncclWindow_t wc, const int64_t* __restrict__ send_counts, int R,
                                 int me) {
  for (int i = threadIdx.x; i < R * R * 2; i += blockDim.x) {  // i = (peer, dst, k)
    const int p = i / (R * 2), rest = i % (R * 2);
    int64_t* dstw = static_cast<int64_t*>(ncclGetLsaPointer(wc, 0, p));
    dstw[(int64_t)me * R * 2 + rest] = send_counts[rest];
  }
  __syncthreads();
  lsa_barrier(dc);
}

// a barrier alone (after a copy kernel: the peers' stores into this rank's windows are
// complete and visible when it returns)
__global__ void ep_barrier_kernel(ncclDevComm dc) { lsa_barrier(dc); }

// kernel 2: x rows and records of every destination block into the destination's windows
__global__ void __launch_bounds__(256)
    ep_dispatch_copy_kernel(ncclWindow_t wc, ncclWindow_t wx, ncclWindow_t wr, const uint4* __restrict__ x_send,
                            const int32_t* __restrict__ rec_send, int R, int me, int64_t row_vec, int64_t row_cap,
                            int64_t rec_cap) {
  __shared__ int64_t send_row[kMaxR + 1], send_rec[kMaxR + 1], roff[kMaxR], qoff[kMaxR];
  const int64_t* c = static_cast<const int64_t*>(ncclGetLocalPointer(wc, 0));
  if (threadIdx.x == 0) {
    send_row[0] = send_rec[0] = 0;
    for (int s = 0; s < R; ++s) {
      send_row[s + 1] = send_row[s] + cnt(c, R, me, s, 0);
      send_rec[s + 1] = send_rec[s] + cnt(c, R, me, s, 1);
      int64_t ro = 0, qo = 0;
      for (int src = 0; src < me; ++src) {
        ro += cnt(c, R, src, s, 0);
        qo += cnt(c, R, src, s, 1);
      }
      roff[s] = ro;  // first row / record of my block in s's windows
      qoff[s] = qo;
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (gridDim.x * (int64_t)blockDim.x) >> 5;
  // rows: one warp per row, 16-byte vectors
  for (int64_t q = gw; q < send_row[R]; q += nw) {
    int s = 0;
    while (s + 1 < R && send_row[s + 1] <= q) ++s;
    const int64_t at = roff[s] + (q - send_row[s]);
    if (at >= row_cap) continue;  // over capacity: dropped (the host checks the counts and raises)
    uint4* dst = static_cast<uint4*>(ncclGetLsaPointer(wx, (size_t)at * row_vec * 16, s));
    const uint4* src = x_send + q * row_vec;
    for (int64_t v = lane; v < row_vec; v += 32) dst[v] = src[v];
  }
  // records: one thread each; the slot becomes the receiver's row index
  const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = gt; q < send_rec[R]; q += nt) {
    int s = 0;
    while (s + 1 < R && send_rec[s + 1] <= q) ++s;
    const int64_t at = qoff[s] + (q - send_rec[s]);
    if (at >= rec_cap) continue;
    int32_t* dst = static_cast<int32_t*>(ncclGetLsaPointer(wr, (size_t)at * 12, s));
    dst[0] = rec_send[3 * q];
    dst[1] = rec_send[3 * q + 1];
    dst[2] = rec_send[3 * q + 2] + (int32_t)roff[s];
  }
}

// kernel 4: the received rows' partial outputs back to their home ranks
__global__ void __launch_bounds__(256)
    ep_return_copy_kernel(ncclWindow_t wc, ncclWindow_t wy, const uint4* __restrict__ y_part, int64_t rows, int R,
                          int me, int64_t row_vec, int64_t row_cap) {
  __shared__ int64_t recv_row[kMaxR + 1], home_off[kMaxR];
  const int64_t* c = static_cast<const int64_t*>(ncclGetLocalPointer(wc, 0));
  if (threadIdx.x == 0) {
    recv_row[0] = 0;
    for (int src = 0; src < R; ++src) {
      recv_row[src + 1] = recv_row[src] + cnt(c, R, src, me, 0);
      int64_t h = 0;
      for (int t = 0; t < me; ++t) h += cnt(c, R, src, t, 0);
      home_off[src] = h;  // first row of src's block for me in src's x_send / y_ret
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (gridDim.x * (int64_t)blockDim.x) >> 5;
  const int64_t n = rows < recv_row[R] ? rows : recv_row[R];
  for (int64_t j = gw; j < n; j += nw) {
    int src = 0;
    while (src + 1 < R && recv_row[src + 1] <= j) ++src;
    const int64_t at = home_off[src] + (j - recv_row[src]);
    if (at >= row_cap) continue;
    uint4* dst = static_cast<uint4*>(ncclGetLsaPointer(wy, (size_t)at * row_vec * 16, src));
    const uint4* s = y_part + j * row_vec;
    for (int64_t v = lane; v < row_vec; v += 32) dst[v] = s[v];
  }
}

int grid_for(int64_t work, int per_block) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t g = (work + per_block - 1) / per_block;
  return (int)(g < 1 ? 1 : (g > 8 * sms ? 8 * sms : g));
}
}  // namespace

extern "C" {

size_t omnimoe_ep_dev_unique_id_bytes(void) { return sizeof(ncclUniqueId); }

omnimoe_status omnimoe_ep_dev_unique_id(void* out) {
  if (!out) return fail("unique_id: null output", OMNIMOE_ERR_INVALID_ARGUMENT);
  ncclUniqueId id;
  EP_NCCL(ncclGetUniqueId(&id));
  memcpy(out, &id, sizeof(id));
  return OMNIMOE_OK;
}

omnimoe_status omnimoe_ep_dev_create(const void* unique_id, int32_t rank, int32_t world, int64_t d, int64_t row_cap,
                                     int64_t rec_cap, omnimoe_ep_comm** out) {
  if (!unique_id || !out || world < 1 || world > kMaxR || rank < 0 || rank >= world || d < 8 || d % 8 ||
      row_cap < 1 || rec_cap < 1)
    return fail("ep_dev_create: need 1 <= world <= 16, 0 <= rank < world, d % 8 == 0, capacities >= 1",
                OMNIMOE_ERR_INVALID_ARGUMENT);
  auto* c = new omnimoe_ep_comm();
  c->rank = rank;
  c->world = world;
  c->d = d;
  c->row_cap = row_cap;
  c->rec_cap = rec_cap;
  ncclUniqueId id;
  memcpy(&id, unique_id, sizeof(id));
  auto cleanup = [&](omnimoe_status s) {
    omnimoe_ep_dev_destroy(c);
    return s;
  };
  if (ncclCommInitRank(&c->comm, world, id, rank) != ncclSuccess)
    return cleanup(fail("ncclCommInitRank failed", OMNIMOE_ERR_CUDA));
  const size_t sz[4] = {(size_t)world * world * 2 * sizeof(int64_t), (size_t)row_cap * d * 2, (size_t)rec_cap * 12,
                        (size_t)row_cap * d * 2};
  void** bufs[4] = {&c->counts, &c->x, &c->rec, &c->y};
  ncclWindow_t* wins[4] = {&c->wc, &c->wx, &c->wr, &c->wy};
  for (int i = 0; i < 4; ++i) {
    const size_t b = (sz[i] + 4095) / 4096 * 4096;
    if (ncclMemAlloc(bufs[i], b) != ncclSuccess) return cleanup(fail("ncclMemAlloc failed", OMNIMOE_ERR_CUDA));
    if (ncclCommWindowRegister(c->comm, *bufs[i], b, wins[i], NCCL_WIN_COLL_SYMMETRIC) != ncclSuccess)
      return cleanup(fail("ncclCommWindowRegister failed", OMNIMOE_ERR_CUDA));
  }
  ncclDevCommRequirements req = {};
  req.lsaBarrierCount = 1;
  if (ncclDevCommCreate(c->comm, &req, &c->dev) != ncclSuccess)
    return cleanup(fail("ncclDevCommCreate failed", OMNIMOE_ERR_CUDA));
  *out = c;
  return OMNIMOE_OK;
}

omnimoe_status omnimoe_ep_dev_destroy(omnimoe_ep_comm* c) {
  if (!c) return OMNIMOE_OK;
  if (c->comm) {
    if (c->dev.windowTable || c->dev.nRanks) ncclDevCommDestroy(c->comm, &c->dev);
    ncclWindow_t wins[4] = {c->wc, c->wx, c->wr, c->wy};
    for (auto w : wins)
      if (w) ncclCommWindowDeregister(c->comm, w);
  }
  void* bufs[4] = {c->counts, c->x, c->rec, c->y};
  for (auto b : bufs)
    if (b) ncclMemFree(b);
  if (c->comm) ncclCommDestroy(c->comm);
  delete c;
  return OMNIMOE_OK;
}

omnimoe_status omnimoe_ep_dev_buffers(const omnimoe_ep_comm* c, void** x_recv, int32_t** rec_recv, void** y_ret,
                                      int64_t** counts) {
  if (!c) return fail("ep_dev_buffers: null comm", OMNIMOE_ERR_INVALID_ARGUMENT);
  if (x_recv) *x_recv = c->x;
  if (rec_recv) *rec_recv = static_cast<int32_t*>(c->rec);
  if (y_ret) *y_ret = c->y;
  if (counts) *counts = static_cast<int64_t*>(c->counts);
  return OMNIMOE_OK;
}

omnimoe_status omnimoe_ep_dev_dispatch(omnimoe_ep_comm* c, const void* x_send, const int32_t* rec_send,
                                       const int64_t* send_counts, omnimoe_stream_t stream) {
  if (!c || !send_counts) return fail("ep_dev_dispatch: null comm / counts", OMNIMOE_ERR_INVALID_ARGUMENT);
  cudaStream_t st = (cudaStream_t)stream;
  const int R = c->world;
  ep_counts_kernel<<<1, 128, 0, st>>>(c->dev, c->wc, send_counts, R, c->rank);
  EP_LAUNCH("ep_counts_kernel");
  // the sizes are on the device; the copy kernel bounds itself by them (capacity-sized grid)
  ep_dispatch_copy_kernel<<<grid_for(c->row_cap * 32, 256), 256, 0, st>>>(
      c->wc, c->wx, c->wr, static_cast<const uint4*>(x_send), rec_send, R, c->rank, c->d * 2 / 16, c->row_cap,
      c->rec_cap);
  EP_LAUNCH("ep_dispatch_copy_kernel");
  ep_barrier_kernel<<<1, 128, 0, st>>>(c->dev);
  EP_LAUNCH("ep_barrier_kernel");
  return OMNIMOE_OK;
}

omnimoe_status omnimoe_ep_dev_return(omnimoe_ep_comm* c, const void* y_part, int64_t rows_recv,
                                     omnimoe_stream_t stream) {
  if (!c || rows_recv < 0 || rows_recv > c->row_cap)
    return fail("ep_dev_return: null comm or rows outside [0, row_cap]", OMNIMOE_ERR_INVALID_ARGUMENT);
  cudaStream_t st = (cudaStream_t)stream;
  if (rows_recv > 0) {
    ep_return_copy_kernel<<<grid_for(rows_recv * 32, 256), 256, 0, st>>>(
        c->wc, c->wy, static_cast<const uint4*>(y_part), rows_recv, c->world, c->rank, c->d * 2 / 16, c->row_cap);
    EP_LAUNCH("ep_return_copy_kernel");
  }
  ep_barrier_kernel<<<1, 128, 0, st>>>(c->dev);
  EP_LAUNCH("ep_barrier_kernel");
  return OMNIMOE_OK;
}

const char* omnimoe_ep_last_error(void) { return g_err.c_str(); }

}  // extern "C"
