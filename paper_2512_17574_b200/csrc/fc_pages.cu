// fc_pages.cu -- NEXT-2, the paged embedding buffer (PAPER.md P:482-502,
// Fig. 10; SPEC embed_buffer S:218-290; reading R21 in DESIGN.md).
//
// Host: the page table (fc_pages_*).  Pages are owned by one request or free;
// each iteration's reads / writes are described by the paper's four indices
// (pv_indptr, pv_page_indptr, pv_page_indices, pv_cu_page_len),
// and pages a read has fully consumed are released eagerly after the
// iteration ("e.g., pages 8 and 11").
//
// Device: fc_paged_copy, read_chunk / write_chunk between the pool and a
// contiguous chunk ("materialise them into contiguous memory only at use
// time").  A request's run of tokens inside one page is contiguous in
// both the pool and the chunk, so the index becomes a list of contiguous
// byte blocks (at most one per page touched) and the kernel is a batched
// memcpy: the blocks are laid end to end in one virtual byte range, every CTA
// takes an equal slice of it and copies with 16-byte (or 8-byte) vector
// loads/stores, 4 in flight per thread.  HBM-bound: 2 x row_bytes per row.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <deque>
#include <new>
#include <set>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "fc.h"
#include "fc_internal.h"
#include "fc_launch.h"

using namespace fc;

// ---------------------------------------------------------------- page table

namespace {

struct Request {
  std::deque<int32_t> pages;  // owned pages in token order; pages[0] holds token `base`
  int64_t base = 0;           // first token of pages[0] (a multiple of page_rows)
  int64_t reserved = 0;       // tokens alloc_pages has made room for
  int64_t written = 0, read = 0;
};

}  // namespace

struct fc_pages_s {
  int64_t total = 0;
  int32_t page_rows = 0;
  std::set<int32_t> free_ids;  // lowest id first
  std::unordered_map<int64_t, Request> reqs;
  std::vector<int32_t> consumed;  // awaiting fc_pages_free_consumed, in consumption order
  int64_t owned = 0;
};

namespace {

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// pages a request holds or held: capacity in tokens
int64_t capacity(const fc_pages_s* t, const Request& r) {
  return r.base + static_cast<int64_t>(r.pages.size()) * t->page_rows;
}

}  // namespace

extern "C" {

fc_status fc_pages_create(int64_t total_pages, int32_t page_rows, fc_pages_t** out) {
  if (!out) return fail(FC_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (total_pages < 0 || total_pages > INT32_MAX) return fail(FC_ERR_INVALID_ARG, "total_pages outside [0, 2^31)");
  if (page_rows <= 0 || page_rows > (1 << 20) || (page_rows & (page_rows - 1)))
    return fail(FC_ERR_INVALID_ARG, "page_rows must be a power of two <= 2^20");
  try {
    auto* t = new fc_pages_s();
    t->total = total_pages;
    t->page_rows = page_rows;
    for (int64_t i = 0; i < total_pages; ++i) t->free_ids.insert(t->free_ids.end(), static_cast<int32_t>(i));
    *out = t;
  } catch (const std::bad_alloc&) {
    return fail(FC_ERR_OOM, "page table allocation");
  }
  return FC_OK;
}

void fc_pages_destroy(fc_pages_t* t) { delete t; }

fc_status fc_pages_alloc(fc_pages_t* t, int64_t req, int64_t tokens, int32_t* new_ids, int32_t cap, int32_t* n_new) {
  if (!t) return fail(FC_ERR_INVALID_ARG, "page table is NULL");
  if (tokens < 0) return fail(FC_ERR_INVALID_ARG, "tokens < 0");
  if (n_new) *n_new = 0;
  auto it = t->reqs.find(req);
  const Request empty;
  const Request& r = it == t->reqs.end() ? empty : it->second;
  const int64_t target = std::max(r.reserved, r.written) + tokens;
  const int64_t need = std::max<int64_t>(0, ceil_div(target, t->page_rows) - ceil_div(capacity(t, r), t->page_rows));
  if (need > static_cast<int64_t>(t->free_ids.size()))
    return fail(FC_ERR_OUT_OF_PAGES, "request " + std::to_string(req) + " needs " + std::to_string(need) +
                                         " pages, " + std::to_string(t->free_ids.size()) + " free");
  if (new_ids && need > cap) return fail(FC_ERR_INVALID_ARG, "new_ids capacity < pages appended");
  try {
    Request& w = t->reqs[req];  // creates the entry on first use
    for (int64_t k = 0; k < need; ++k) {
      const int32_t id = *t->free_ids.begin();
      t->free_ids.erase(t->free_ids.begin());
      w.pages.push_back(id);
      if (new_ids) new_ids[k] = id;
    }
    w.reserved = target;
  } catch (const std::bad_alloc&) {
    return fail(FC_ERR_OOM, "page table growth");
  }
  t->owned += need;
  if (n_new) *n_new = static_cast<int32_t>(need);
  return FC_OK;
}

fc_status fc_pages_index(fc_pages_t* t, fc_page_op op, const int64_t* reqs, const int64_t* counts, int32_t n,
                         int64_t* pv_indptr, int32_t* pv_page_indptr, int32_t* pv_page_indices, int32_t cap,
                         int64_t* pv_cu_page_len, int32_t* num_indices) {
  if (!t || n < 0 || (n > 0 && (!reqs || !counts)) || !pv_indptr || !pv_page_indptr || !num_indices ||
      (n > 0 && !pv_cu_page_len) || (op != FC_PAGE_WRITE && op != FC_PAGE_READ))
    return fail(FC_ERR_INVALID_ARG, "fc_pages_index: NULL or out-of-range argument");
  const int64_t P = t->page_rows;
  // validate everything and size the output before any state changes
  std::unordered_set<int64_t> seen;
  int64_t pages = 0;
  for (int32_t i = 0; i < n; ++i) {
    if (counts[i] < 0) return fail(FC_ERR_INVALID_ARG, "counts[" + std::to_string(i) + "] < 0");
    if (!seen.insert(reqs[i]).second)
      return fail(FC_ERR_INVALID_ARG, "request " + std::to_string(reqs[i]) + " appears twice in one index");
    auto it = t->reqs.find(reqs[i]);
    if (it == t->reqs.end()) {
      if (counts[i] == 0) continue;
      return fail(FC_ERR_INVALID_ARG, "request " + std::to_string(reqs[i]) + " has no pages");
    }
    const Request& r = it->second;
    const int64_t cu = op == FC_PAGE_WRITE ? r.written : r.read;
    if (op == FC_PAGE_WRITE && cu + counts[i] > capacity(t, r))
      return fail(FC_ERR_INVALID_ARG, "write past the pages allocated to request " + std::to_string(reqs[i]) +
                                          " (CapacityError)");
    if (op == FC_PAGE_READ && cu + counts[i] > r.written)
      return fail(FC_ERR_INVALID_ARG, "read past the tokens written by request " + std::to_string(reqs[i]) +
                                          " (UnwrittenRange)");
    if (counts[i] > 0) pages += (cu + counts[i] - 1) / P - cu / P + 1;
  }
  *num_indices = static_cast<int32_t>(std::min<int64_t>(pages, INT32_MAX));
  if (pages > cap || (pages > 0 && !pv_page_indices))
    return fail(FC_ERR_INVALID_ARG, "pv_page_indices capacity " + std::to_string(cap) + " < " +
                                        std::to_string(pages) + " pages needed");
  int64_t rows = 0;
  int32_t k = 0;
  pv_indptr[0] = 0;
  pv_page_indptr[0] = 0;
  for (int32_t i = 0; i < n; ++i) {
    auto it = t->reqs.find(reqs[i]);
    if (it == t->reqs.end()) {  // an unknown request with nothing to move
      pv_cu_page_len[i] = 0;
      pv_indptr[i + 1] = rows;
      pv_page_indptr[i + 1] = k;
      continue;
    }
    Request& r = it->second;
    int64_t& cu = op == FC_PAGE_WRITE ? r.written : r.read;
    pv_cu_page_len[i] = cu;
    if (counts[i] > 0) {
      const int64_t g0 = cu / P, g1 = (cu + counts[i] - 1) / P;  // pages holding the first / last token
      for (int64_t g = g0; g <= g1; ++g) pv_page_indices[k++] = r.pages[static_cast<size_t>(g - r.base / P)];
    }
    cu += counts[i];
    rows += counts[i];
    pv_indptr[i + 1] = rows;
    pv_page_indptr[i + 1] = k;
    if (op == FC_PAGE_READ) {  // pages whose last token is now read are consumed
      while (!r.pages.empty() && r.base + P <= r.read) {
        t->consumed.push_back(r.pages.front());
        r.pages.pop_front();
        r.base += P;
        --t->owned;
      }
    }
  }
  return FC_OK;
}

fc_status fc_pages_free_consumed(fc_pages_t* t, int32_t* freed, int32_t cap, int32_t* n_freed) {
  if (!t) return fail(FC_ERR_INVALID_ARG, "page table is NULL");
  const size_t m = t->consumed.size();
  if (freed)
    for (size_t i = 0; i < m && static_cast<int64_t>(i) < cap; ++i) freed[i] = t->consumed[i];
  for (int32_t id : t->consumed) t->free_ids.insert(id);
  t->consumed.clear();
  if (n_freed) *n_freed = static_cast<int32_t>(m);
  return FC_OK;
}

fc_status fc_pages_release(fc_pages_t* t, int64_t req) {
  if (!t) return fail(FC_ERR_INVALID_ARG, "page table is NULL");
  auto it = t->reqs.find(req);
  if (it == t->reqs.end()) return fail(FC_ERR_INVALID_ARG, "unknown request " + std::to_string(req));
  for (int32_t id : it->second.pages) t->consumed.push_back(id);
  t->owned -= static_cast<int64_t>(it->second.pages.size());
  t->reqs.erase(it);
  return FC_OK;
}

fc_status fc_pages_stats(const fc_pages_t* t, int64_t* free_pages, int64_t* owned_pages, int64_t* consumed_pages,
                         int64_t* live_requests) {
  if (!t) return fail(FC_ERR_INVALID_ARG, "page table is NULL");
  if (free_pages) *free_pages = static_cast<int64_t>(t->free_ids.size());
  if (owned_pages) *owned_pages = t->owned;
  if (consumed_pages) *consumed_pages = static_cast<int64_t>(t->consumed.size());
  if (live_requests) *live_requests = static_cast<int64_t>(t->reqs.size());
  return FC_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- device copy

namespace fc {
namespace {

constexpr int kCopyThreads = 256;
constexpr int kCopyUnroll = 4;  // vectors in flight per thread
constexpr int kInlineBlocks = 320;  // blocks carried in the kernel parameters (no upload)

// Block k: bytes [start[k], start[k+1]) of the virtual range are bytes
// [0, len) of pool + pool_off[k] and chunk + chunk_off[k].
struct CopyParams {
  uint8_t* pool;
  uint8_t* chunk;
  const long long* start;  // nblocks + 1 (device descriptor), or null: use the inline arrays
  const long long* pool_off;
  const long long* chunk_off;
  long long total;  // bytes
  int nblocks;
  int read;  // 1: pool -> chunk
  long long istart[kInlineBlocks + 1];
  long long ipool[kInlineBlocks];
  long long ichunk[kInlineBlocks];
};

template <int VEC>
struct Vec;
template <>
struct Vec<16> {
  using T = uint4;
};
template <>
struct Vec<8> {
  using T = uint2;
};

template <int VEC>
__device__ __forceinline__ typename Vec<VEC>::T ld_stream(const void* p) {
  typename Vec<VEC>::T v;
  if constexpr (VEC == 16)
    asm volatile("ld.global.cs.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  else
    asm volatile("ld.global.cs.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}
template <int VEC>
__device__ __forceinline__ void st_stream(void* p, const typename Vec<VEC>::T& v) {
  if constexpr (VEC == 16)
    asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
  else
    asm volatile("st.global.cs.v2.u32 [%0], {%1, %2};" ::"l"(p), "r"(v.x), "r"(v.y) : "memory");
}

template <int VEC>
__global__ void __launch_bounds__(kCopyThreads) fc_paged_copy_kernel(const __grid_constant__ CopyParams p) {
  const long long* start = p.start ? p.start : p.istart;
  const long long* poff = p.start ? p.pool_off : p.ipool;
  const long long* coff = p.start ? p.chunk_off : p.ichunk;
  // this CTA's slice of the virtual range, in whole vectors
  const long long nvec = p.total / VEC;
  const long long v0 = nvec * blockIdx.x / gridDim.x, v1 = nvec * (blockIdx.x + 1) / gridDim.x;
  if (v0 >= v1) return;
  // first block overlapping the slice (largest k with start[k] <= v0 * VEC)
  int lo = 0, hi = p.nblocks - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (start[mid] <= v0 * VEC)
      lo = mid;
    else
      hi = mid - 1;
  }
  for (int k = lo; k < p.nblocks && start[k] < v1 * VEC; ++k) {
    const long long b0 = max(start[k], v0 * VEC), b1 = min(start[k + 1], v1 * VEC);
    const uint8_t* src = (p.read ? p.pool + poff[k] : p.chunk + coff[k]) - start[k];
    uint8_t* dst = (p.read ? p.chunk + coff[k] : p.pool + poff[k]) - start[k];
    long long b = b0 + static_cast<long long>(threadIdx.x) * VEC;
    constexpr long long kStep = static_cast<long long>(kCopyThreads) * VEC;
    for (; b + (kCopyUnroll - 1) * kStep < b1; b += kCopyUnroll * kStep) {
      typename Vec<VEC>::T v[kCopyUnroll];
#pragma unroll
      for (int u = 0; u < kCopyUnroll; ++u) v[u] = ld_stream<VEC>(src + b + u * kStep);
#pragma unroll
      for (int u = 0; u < kCopyUnroll; ++u) st_stream<VEC>(dst + b + u * kStep, v[u]);
    }
    for (; b < b1; b += kStep) st_stream<VEC>(dst + b, ld_stream<VEC>(src + b));
  }
}

}  // namespace
}  // namespace fc

extern "C" fc_status fc_paged_copy(fc_page_op op, const fc_ragged_index* idx, void* pool, int64_t pool_pages,
                                   int32_t page_rows, int64_t row_bytes, void* chunk, void* stream) {
  if (!idx || (op != FC_PAGE_WRITE && op != FC_PAGE_READ))
    return fail(FC_ERR_INVALID_ARG, "fc_paged_copy: NULL index or bad op");
  const int32_t n = idx->num_requests;
  if (n < 0 || (n > 0 && (!idx->pv_indptr || !idx->pv_page_indptr || !idx->pv_cu_page_len)))
    return fail(FC_ERR_INVALID_ARG, "fc_paged_copy: index arrays are NULL");
  if (page_rows <= 0 || (page_rows & (page_rows - 1)) || pool_pages < 0)
    return fail(FC_ERR_INVALID_ARG, "page_rows must be a power of two, pool_pages >= 0");
  if (row_bytes <= 0 || row_bytes % 8) return fail(FC_ERR_INVALID_ARG, "row_bytes must be a positive multiple of 8");
  if (n == 0) return FC_OK;
  if (idx->pv_indptr[0] != 0 || idx->pv_page_indptr[0] != 0)
    return fail(FC_ERR_INVALID_ARG, "pv_indptr[0] and pv_page_indptr[0] must be 0");
  // validate and cut the index into contiguous blocks (one per page touched)
  std::vector<long long> start{0}, poff, coff;
  try {
    for (int32_t i = 0; i < n; ++i) {
      const int64_t c = idx->pv_indptr[i + 1] - idx->pv_indptr[i];
      const int32_t np = idx->pv_page_indptr[i + 1] - idx->pv_page_indptr[i];
      const int64_t cu = idx->pv_cu_page_len[i];
      if (c < 0 || np < 0 || cu < 0)
        return fail(FC_ERR_INVALID_ARG, "request " + std::to_string(i) + ": decreasing indptr or negative cu_page_len");
      const int64_t off = cu % page_rows;
      const int64_t need = c > 0 ? (off + c - 1) / page_rows + 1 : 0;
      if (np < need)
        return fail(FC_ERR_INVALID_ARG, "request " + std::to_string(i) + ": " + std::to_string(np) + " pages for " +
                                            std::to_string(need) + " needed");
      if (c > 0 && !idx->pv_page_indices) return fail(FC_ERR_INVALID_ARG, "pv_page_indices is NULL");
      for (int64_t t = 0, s = off; t < c;) {
        const int32_t page = idx->pv_page_indices[idx->pv_page_indptr[i] + s / page_rows];
        if (page < 0 || page >= pool_pages)
          return fail(FC_ERR_INVALID_ARG, "request " + std::to_string(i) + ": page id " + std::to_string(page) +
                                              " outside the pool");
        const int64_t len = std::min<int64_t>(page_rows - s % page_rows, c - t);
        poff.push_back((static_cast<long long>(page) * page_rows + s % page_rows) * row_bytes);
        coff.push_back((idx->pv_indptr[i] + t) * row_bytes);
        start.push_back(start.back() + len * row_bytes);
        t += len;
        s += len;
      }
    }
  } catch (const std::bad_alloc&) {
    return fail(FC_ERR_OOM, "fc_paged_copy block list");
  }
  const long long total = start.back();
  if (total == 0) return FC_OK;
  if (!pool || !chunk) return fail(FC_ERR_INVALID_ARG, "pool/chunk is NULL");
  if ((reinterpret_cast<uintptr_t>(pool) | reinterpret_cast<uintptr_t>(chunk)) & 15)
    return fail(FC_ERR_INVALID_ARG, "pool and chunk must be 16-byte aligned");
  int dev = 0, major = 0, max_smem = 0, nsm = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  device_attrs(dev, &major, &max_smem, &nsm);
  if (major != 10) return fail(FC_ERR_CUDA, "fc kernels are built for sm_100a only (no CPU/other-arch fallback)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  static thread_local CopyParams prm;
  prm.pool = static_cast<uint8_t*>(pool);
  prm.chunk = static_cast<uint8_t*>(chunk);
  prm.total = total;
  prm.nblocks = static_cast<int>(poff.size());
  prm.read = op == FC_PAGE_READ;
  void* desc = nullptr;
  if (prm.nblocks <= kInlineBlocks) {
    prm.start = prm.pool_off = prm.chunk_off = nullptr;
    std::copy(start.begin(), start.end(), prm.istart);
    std::copy(poff.begin(), poff.end(), prm.ipool);
    std::copy(coff.begin(), coff.end(), prm.ichunk);
  } else {  // descriptor [start | pool_off | chunk_off], stream-ordered, freed after the launch
    const size_t m = poff.size();
    std::vector<long long> host(3 * m + 1);
    std::copy(start.begin(), start.end(), host.begin());
    std::copy(poff.begin(), poff.end(), host.begin() + m + 1);
    std::copy(coff.begin(), coff.end(), host.begin() + 2 * m + 1);
    const size_t bytes = host.size() * sizeof(long long);
    cudaMemPool_t mp = descriptor_pool(dev);
    e = mp ? cudaMallocFromPoolAsync(&desc, bytes, mp, s) : cudaMallocAsync(&desc, bytes, s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync (paged copy descriptor)");
    e = cudaMemcpyAsync(desc, host.data(), bytes, cudaMemcpyHostToDevice, s);  // pageable: staged before return
    if (e != cudaSuccess) {
      cudaFreeAsync(desc, s);
      return cuda_fail(e, "paged copy descriptor upload");
    }
    prm.start = static_cast<const long long*>(desc);
    prm.pool_off = prm.start + m + 1;
    prm.chunk_off = prm.start + 2 * m + 1;
  }
  // 8 CTAs of 256 threads per SM, fewer for a small chunk (>= 16 KB per CTA).
  // A/B (round 2, cold single launches under ncu): ld/st .cs vs .nc / write-back,
  // 4 / 8 / 16 CTAs per SM, 4 / 8 vectors in flight: all within 3%.
  const int grid = static_cast<int>(std::max<long long>(1, std::min<long long>(static_cast<long long>(nsm) * 8,
                                                                               total / 16384)));
  if (row_bytes % 16 == 0)
    fc_paged_copy_kernel<16><<<grid, kCopyThreads, 0, s>>>(prm);
  else
    fc_paged_copy_kernel<8><<<grid, kCopyThreads, 0, s>>>(prm);
  e = cudaGetLastError();
  if (desc) cudaFreeAsync(desc, s);
  if (e != cudaSuccess) return cuda_fail(e, "paged copy launch");
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  return FC_OK;
}
