// fc_gather.cpp -- the exchange step of the path (a10): the row shards of
// all ranks are assembled on the encoder GPU ("collective
// scatter" into the IPC patch buffer, "NCCL ... for IPC buffer
// transfers"; reading R9).  Rows are t-major, so every rank owns ONE
// contiguous row range and the exchange is a gatherv: NCCL has no gatherv,
// so it is a grouped ncclSend/ncclRecv with the encoder receiving each peer's
// shard directly at full + row_begin*1176 (no staging copy).
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "fc_internal.h"

using namespace fc;

static fc_status nccl_fail(ncclResult_t r, const char* what) {
  return fail(FC_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

extern "C" {

fc_status fc_nccl_unique_id(uint8_t id[128]) {
  if (!id) return fail(FC_ERR_INVALID_ARG, "id is NULL");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId u;
  ncclResult_t r = ncclGetUniqueId(&u);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(id, &u, 128);
  return FC_OK;
}

fc_status fc_nccl_comm_init(const uint8_t id[128], int32_t world_size, int32_t rank, void** comm) {
  if (!id || !comm) return fail(FC_ERR_INVALID_ARG, "id/comm is NULL");
  if (rank < 0 || rank >= world_size) return fail(FC_ERR_RANK, "rank outside [0, world_size)");
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  ncclComm_t c = nullptr;
  ncclResult_t r = ncclCommInitRank(&c, world_size, u, rank);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
  *comm = c;
  return FC_OK;
}

fc_status fc_nccl_comm_destroy(void* comm) {
  if (!comm) return FC_OK;
  ncclResult_t r = ncclCommDestroy(static_cast<ncclComm_t>(comm));
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommDestroy");
  return FC_OK;
}

// ---------------------------------------------------------------- CUDA IPC
static fc_status cuda_err(cudaError_t e, const char* what) {
  return fail(FC_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

fc_status fc_ipc_export(void* dev_ptr, uint8_t handle[64]) {
  if (!dev_ptr || !handle) return fail(FC_ERR_INVALID_ARG, "dev_ptr/handle is NULL");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t size");
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, dev_ptr);
  if (e != cudaSuccess) return cuda_err(e, "cudaIpcGetMemHandle");
  std::memcpy(handle, &h, 64);
  return FC_OK;
}

fc_status fc_ipc_export_range(void* ptr, uint8_t handle[64], int64_t* offset) {
  if (!ptr || !handle || !offset) return fail(FC_ERR_INVALID_ARG, "ptr/handle/offset is NULL");
  CUdeviceptr base = 0;
  size_t size = 0;
  // the runtime has no base-address query; the driver's cuMemGetAddressRange does
  using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static GetRange fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<GetRange>(nullptr);
    return reinterpret_cast<GetRange>(f);
  }();
  if (!fn) return fail(FC_ERR_CUDA, "cuMemGetAddressRange unavailable");
  if (fn(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS)
    return fail(FC_ERR_INVALID_ARG, "ptr is not device memory of this process");
  *offset = static_cast<int64_t>(reinterpret_cast<CUdeviceptr>(ptr) - base);
  return fc_ipc_export(reinterpret_cast<void*>(base), handle);
}

fc_status fc_ipc_import(const uint8_t handle[64], void** dev_ptr) {
  if (!handle || !dev_ptr) return fail(FC_ERR_INVALID_ARG, "handle/dev_ptr is NULL");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  const cudaError_t e = cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return cuda_err(e, "cudaIpcOpenMemHandle");
  return FC_OK;
}

fc_status fc_ipc_close(void* dev_ptr) {
  if (!dev_ptr) return fail(FC_ERR_INVALID_ARG, "dev_ptr is NULL");
  const cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
  if (e != cudaSuccess) return cuda_err(e, "cudaIpcCloseMemHandle");
  return FC_OK;
}

// The transfers of one rank's part of an exchange (R9 gather / NEXT-1 column
// split), in bytes; fc_gather and fc_scatter_columns execute exactly this list.
static fc_status schedule(const fc_plan_t* P, int32_t rank, fc_exchange_kind kind, std::vector<fc_transfer>* out) {
  out->clear();
  if (!P) return fail(FC_ERR_INVALID_ARG, "plan is NULL");
  if (rank < 0 || rank >= P->world) return fail(FC_ERR_RANK, "rank outside [0, world_size)");
  const fc_rank_plan& me = P->ranks[rank].p;
  const int64_t my_rows = me.row_end - me.row_begin;
  if (kind == FC_XCHG_GATHER) {
    // rows are exchanged as bytes: 1176 tokens x (4 B fp32 | 2 B bf16 | 1 B u8 code)
    const int elem = P->cfg.token_dtype == FC_TOKENS_U8 ? 1 : P->cfg.token_dtype == FC_TOKENS_BF16 ? 2 : 4;
    const int64_t rb = static_cast<int64_t>(kCols) * elem;
    const int e = P->cfg.encoder_rank;
    if (rank == e) {
      if (my_rows) out->push_back({rank, FC_XFER_LOCAL, 0, me.row_begin * rb, my_rows * rb});
      for (int p = 0; p < P->world; ++p) {
        const fc_rank_plan& rp = P->ranks[p].p;
        if (p != e && rp.row_end > rp.row_begin)
          out->push_back({p, FC_XFER_RECV, 0, rp.row_begin * rb, (rp.row_end - rp.row_begin) * rb});
      }
    } else if (my_rows) {
      out->push_back({e, FC_XFER_SEND, 0, 0, my_rows * rb});
    }
    return FC_OK;
  }
  if (kind != FC_XCHG_COLSPLIT) return fail(FC_ERR_INVALID_ARG, "unknown exchange kind");
  if (kCols % P->world != 0) return fail(FC_ERR_UNSUPPORTED, "column split: world_size must divide 1176");
  // blocks [W][my_rows][C] fp32 -> mine [token_rows][C]: block p of my rows goes
  // to rank p; rank p's block `rank` lands at mine + row_begin_p * C
  const int64_t cb = static_cast<int64_t>(kCols / P->world) * 4;  // bytes per row of a block
  if (my_rows) out->push_back({rank, FC_XFER_LOCAL, rank * my_rows * cb, me.row_begin * cb, my_rows * cb});
  for (int p = 0; p < P->world; ++p) {
    if (p == rank) continue;
    const fc_rank_plan& rp = P->ranks[p].p;
    if (my_rows) out->push_back({p, FC_XFER_SEND, p * my_rows * cb, 0, my_rows * cb});
    if (rp.row_end > rp.row_begin)
      out->push_back({p, FC_XFER_RECV, 0, rp.row_begin * cb, (rp.row_end - rp.row_begin) * cb});
  }
  return FC_OK;
}

// Run a schedule: local copies on the stream, sends/receives as one NCCL group.
static fc_status run_schedule(const std::vector<fc_transfer>& xs, int world, void* comm, const void* src, void* dst,
                              void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint8_t* sb = static_cast<const uint8_t*>(src);
  uint8_t* db = static_cast<uint8_t*>(dst);
  for (const fc_transfer& x : xs)
    if (x.dir == FC_XFER_LOCAL && db + x.dst_offset != sb + x.src_offset) {
      cudaError_t ce = cudaMemcpyAsync(db + x.dst_offset, sb + x.src_offset, static_cast<size_t>(x.bytes),
                                       cudaMemcpyDeviceToDevice, s);
      if (ce != cudaSuccess) return fail(FC_ERR_CUDA, std::string("local shard copy: ") + cudaGetErrorString(ce));
    }
  if (world == 1) return FC_OK;
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  ncclResult_t r = ncclGroupStart();
  if (r != ncclSuccess) return nccl_fail(r, "ncclGroupStart");
  for (const fc_transfer& x : xs) {
    if (x.dir == FC_XFER_SEND) r = ncclSend(sb + x.src_offset, static_cast<size_t>(x.bytes), ncclUint8, x.peer, c, s);
    if (x.dir == FC_XFER_RECV) r = ncclRecv(db + x.dst_offset, static_cast<size_t>(x.bytes), ncclUint8, x.peer, c, s);
    if (r != ncclSuccess) break;
  }
  ncclResult_t r2 = ncclGroupEnd();
  if (r != ncclSuccess) return nccl_fail(r, "ncclSend/ncclRecv");
  if (r2 != ncclSuccess) return nccl_fail(r2, "ncclGroupEnd");
  return FC_OK;
}

fc_status fc_exchange_schedule(const fc_plan_t* P, int32_t rank, fc_exchange_kind kind, fc_transfer* out,
                               int32_t capacity, int32_t* count) {
  if (!count) return fail(FC_ERR_INVALID_ARG, "count is NULL");
  std::vector<fc_transfer> xs;
  const fc_status st = schedule(P, rank, kind, &xs);
  if (st != FC_OK) return st;
  *count = static_cast<int32_t>(xs.size());
  if (static_cast<int32_t>(xs.size()) > capacity || (!out && !xs.empty()))
    return out ? fail(FC_ERR_INVALID_ARG, "transfer array too short (count holds the size needed)") : FC_OK;
  std::copy(xs.begin(), xs.end(), out);
  return FC_OK;
}

fc_status fc_gather(const fc_plan_t* P, int32_t rank, void* comm, const void* shard, void* full, void* stream) {
  NvtxRange nvtx("fc_gather");
  std::vector<fc_transfer> xs;
  fc_status st = schedule(P, rank, FC_XCHG_GATHER, &xs);
  if (st != FC_OK) return st;
  const fc_rank_plan& me = P->ranks[rank].p;
  if (rank == P->cfg.encoder_rank && !full) return fail(FC_ERR_INVALID_ARG, "encoder rank needs the full buffer");
  if (me.row_end > me.row_begin && !shard) return fail(FC_ERR_INVALID_ARG, "shard is NULL");
  if (P->world > 1 && !comm) return fail(FC_ERR_INVALID_ARG, "comm is NULL with world_size > 1");
  return run_schedule(xs, P->world, comm, shard, full, stream);
}

fc_status fc_scatter_columns(const fc_plan_t* P, int32_t rank, void* comm, const float* blocks, float* mine,
                             void* stream) {
  std::vector<fc_transfer> xs;
  fc_status st = schedule(P, rank, FC_XCHG_COLSPLIT, &xs);
  if (st != FC_OK) return st;
  if (!mine) return fail(FC_ERR_INVALID_ARG, "mine is NULL");
  const fc_rank_plan& me = P->ranks[rank].p;
  if (me.row_end > me.row_begin && !blocks) return fail(FC_ERR_INVALID_ARG, "blocks is NULL");
  if (P->world > 1 && !comm) return fail(FC_ERR_INVALID_ARG, "comm is NULL with world_size > 1");
  return run_schedule(xs, P->world, comm, blocks, mine, stream);
}

}  // extern "C"
