// fc_gather.cpp -- the exchange step of the path (a10): the row shards of
// all ranks are assembled on the encoder GPU ("collective
// scatter" into the IPC patch buffer, "NCCL ... for IPC buffer
// transfers"; reading R9).  Rows are t-major, so every rank owns ONE
// contiguous row range and the exchange is a gatherv: NCCL has no gatherv,
// so it is a grouped ncclSend/ncclRecv with the encoder receiving each peer's
// shard directly at full + row_begin*1176 (no staging copy).
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstring>
#include <string>

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

fc_status fc_gather(const fc_plan_t* P, int32_t rank, void* comm, const void* shard, void* full, void* stream) {
  if (!P) return fail(FC_ERR_INVALID_ARG, "plan is NULL");
  if (rank < 0 || rank >= P->world) return fail(FC_ERR_RANK, "rank outside [0, world_size)");
  const int e = P->cfg.encoder_rank;
  const fc_rank_plan& me = P->ranks[rank].p;
  // rows are exchanged as bytes: 1176 tokens x (4 B fp32 | 2 B bf16 | 1 B u8 code)
  const int elem = P->cfg.token_dtype == FC_TOKENS_U8 ? 1 : P->cfg.token_dtype == FC_TOKENS_BF16 ? 2 : 4;
  const size_t row_bytes = static_cast<size_t>(kCols) * elem;
  const size_t my_bytes = static_cast<size_t>(me.row_end - me.row_begin) * row_bytes;
  uint8_t* fullb = static_cast<uint8_t*>(full);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (rank == e && !full) return fail(FC_ERR_INVALID_ARG, "encoder rank needs the full buffer");
  if (my_bytes && !shard) return fail(FC_ERR_INVALID_ARG, "shard is NULL");
  if (P->world > 1 && !comm) return fail(FC_ERR_INVALID_ARG, "comm is NULL with world_size > 1");
  if (rank == e && my_bytes) {
    uint8_t* dst = fullb + static_cast<size_t>(me.row_begin) * row_bytes;
    if (dst != shard) {
      cudaError_t ce = cudaMemcpyAsync(dst, shard, my_bytes, cudaMemcpyDeviceToDevice, s);
      if (ce != cudaSuccess) return fail(FC_ERR_CUDA, std::string("own shard copy: ") + cudaGetErrorString(ce));
    }
  }
  if (P->world == 1) return FC_OK;
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  ncclResult_t r = ncclGroupStart();
  if (r != ncclSuccess) return nccl_fail(r, "ncclGroupStart");
  if (rank == e) {
    for (int p = 0; p < P->world; ++p) {
      if (p == e) continue;
      const fc_rank_plan& rp = P->ranks[p].p;
      const size_t n = static_cast<size_t>(rp.row_end - rp.row_begin) * row_bytes;
      if (!n) continue;
      r = ncclRecv(fullb + static_cast<size_t>(rp.row_begin) * row_bytes, n, ncclUint8, p, c, s);
      if (r != ncclSuccess) break;
    }
  } else if (my_bytes) {
    r = ncclSend(shard, my_bytes, ncclUint8, e, c, s);
  }
  ncclResult_t r2 = ncclGroupEnd();
  if (r != ncclSuccess) return nccl_fail(r, "ncclSend/ncclRecv");
  if (r2 != ncclSuccess) return nccl_fail(r2, "ncclGroupEnd");
  return FC_OK;
}

fc_status fc_scatter_columns(const fc_plan_t* P, int32_t rank, void* comm, const float* blocks, float* mine,
                             void* stream) {
  if (!P) return fail(FC_ERR_INVALID_ARG, "plan is NULL");
  if (rank < 0 || rank >= P->world) return fail(FC_ERR_RANK, "rank outside [0, world_size)");
  if (kCols % P->world != 0) return fail(FC_ERR_UNSUPPORTED, "column split: world_size must divide 1176");
  if (!mine) return fail(FC_ERR_INVALID_ARG, "mine is NULL");
  const size_t C = static_cast<size_t>(kCols / P->world);
  const fc_rank_plan& me = P->ranks[rank].p;
  const size_t my_rows = static_cast<size_t>(me.row_end - me.row_begin);
  if (my_rows && !blocks) return fail(FC_ERR_INVALID_ARG, "blocks is NULL");
  if (P->world > 1 && !comm) return fail(FC_ERR_INVALID_ARG, "comm is NULL with world_size > 1");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // own block: rows [row_begin, row_end) of this rank's column slice
  if (my_rows) {
    cudaError_t ce = cudaMemcpyAsync(mine + static_cast<size_t>(me.row_begin) * C, blocks + rank * my_rows * C,
                                     my_rows * C * sizeof(float), cudaMemcpyDeviceToDevice, s);
    if (ce != cudaSuccess) return fail(FC_ERR_CUDA, std::string("own block copy: ") + cudaGetErrorString(ce));
  }
  if (P->world == 1) return FC_OK;
  // all-to-all: block p of my rows -> rank p; rank p's block `rank` -> my rows [row_begin_p, row_end_p)
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  ncclResult_t r = ncclGroupStart();
  if (r != ncclSuccess) return nccl_fail(r, "ncclGroupStart");
  for (int p = 0; p < P->world && r == ncclSuccess; ++p) {
    if (p == rank) continue;
    const fc_rank_plan& rp = P->ranks[p].p;
    const size_t prow = static_cast<size_t>(rp.row_end - rp.row_begin);
    if (my_rows) r = ncclSend(blocks + p * my_rows * C, my_rows * C, ncclFloat32, p, c, s);
    if (r == ncclSuccess && prow)
      r = ncclRecv(mine + static_cast<size_t>(rp.row_begin) * C, prow * C, ncclFloat32, p, c, s);
  }
  ncclResult_t r2 = ncclGroupEnd();
  if (r != ncclSuccess) return nccl_fail(r, "ncclSend/ncclRecv");
  if (r2 != ncclSuccess) return nccl_fail(r2, "ncclGroupEnd");
  return FC_OK;
}

}  // extern "C"
