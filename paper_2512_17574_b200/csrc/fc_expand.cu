// fc_expand.cu -- fc_expand_tokens: u8 codes -> fp32 / bf16 tokens (R5 on the
// NEXT-1 exchange format).  A multi-GPU request gathers 1176-byte code rows
// instead of 4704-byte token rows; the encoder GPU then expands them here.
//
// Pure streaming kernel, HBM-bound: per token row 1176 B read, 4704 B (fp32)
// or 2352 B (bf16) written.  Columns are (c, tp, ph, pw), so a unit of 4
// consecutive columns (392 = 98 * 4 per channel) has one channel: each thread
// loads 4 codes (4 B), looks them up in the channel's 256-entry table (smem)
// and writes 4 tokens with one streaming vector store.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <string>

#include "fc.h"
#include "fc_internal.h"

namespace fc {

namespace {

constexpr int kUnitsPerRow = kCols / 4;  // 294 units of 4 codes; 392 = 98 * 4 per channel
constexpr int kThreadsX = 256;
constexpr int kUnroll = 4;  // units in flight per thread (memory-level parallelism)

struct ExpandParams {
  const uint32_t* codes;  // rows x 294 units of 4 codes
  void* tokens;
  long long units;        // rows * 294
  uint32_t lut[768];      // token bits per (channel, code): fp32 bits or bf16 bits
};

// One unit = 4 consecutive codes (4 B) -> 4 tokens (16 B fp32 / 8 B bf16).  A
// warp's loads cover 128 contiguous bytes and each of its store instructions
// 512 (fp32) or 256 (bf16) contiguous bytes: whole sectors, no partial writes.
template <int TOK>
__device__ __forceinline__ void expand_unit(const uint32_t* lut, void* tokens, long long u, uint32_t c) {
  const uint32_t* t = lut + (static_cast<int>(u % kUnitsPerRow) / 98) * 256;
  const uint32_t v0 = t[c & 0xFF], v1 = t[(c >> 8) & 0xFF], v2 = t[(c >> 16) & 0xFF], v3 = t[c >> 24];
  if constexpr (TOK == FC_TOKENS_BF16) {
    uint2* dst = static_cast<uint2*>(tokens) + u;
    asm volatile("st.global.cs.v2.u32 [%0], {%1, %2};" ::"l"(dst), "r"(v0 | (v1 << 16)), "r"(v2 | (v3 << 16))
                 : "memory");
  } else {
    uint4* dst = static_cast<uint4*>(tokens) + u;
    asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "r"(v0), "r"(v1), "r"(v2), "r"(v3)
                 : "memory");
  }
}

template <int TOK>
__global__ void __launch_bounds__(kThreadsX) fc_expand_kernel(const __grid_constant__ ExpandParams p) {
  __shared__ uint32_t lut[768];
  for (int i = threadIdx.x; i < 768; i += kThreadsX) lut[i] = p.lut[i];
  __syncthreads();
  const long long stride = static_cast<long long>(gridDim.x) * kThreadsX;
  long long u = static_cast<long long>(blockIdx.x) * kThreadsX + threadIdx.x;
  for (; u + (kUnroll - 1) * stride < p.units; u += kUnroll * stride) {
    uint32_t c[kUnroll];
#pragma unroll
    for (int k = 0; k < kUnroll; ++k)
      asm volatile("ld.global.cs.u32 %0, [%1];" : "=r"(c[k]) : "l"(p.codes + u + k * stride));
#pragma unroll
    for (int k = 0; k < kUnroll; ++k) expand_unit<TOK>(lut, p.tokens, u + k * stride, c[k]);
  }
  for (; u < p.units; u += stride) {  // tail
    uint32_t c;
    asm volatile("ld.global.cs.u32 %0, [%1];" : "=r"(c) : "l"(p.codes + u));
    expand_unit<TOK>(lut, p.tokens, u, c);
  }
}

}  // namespace

std::atomic<uint64_t>& launch_counter();

}  // namespace fc

using namespace fc;

extern "C" fc_status fc_expand_tokens(const fc_plan_t* P, int64_t rows, const uint8_t* codes, void* tokens,
                                      fc_token_dtype out_dtype, void* stream) {
  if (!P) return fail(FC_ERR_INVALID_ARG, "plan is NULL");
  if (rows < 0) return fail(FC_ERR_INVALID_ARG, "rows < 0");
  if (out_dtype != FC_TOKENS_F32 && out_dtype != FC_TOKENS_BF16)
    return fail(FC_ERR_UNSUPPORTED, "fc_expand_tokens writes F32 or BF16 tokens");
  if (rows == 0) return FC_OK;
  if (!codes || !tokens) return fail(FC_ERR_INVALID_ARG, "codes/tokens is NULL");
  if ((reinterpret_cast<uintptr_t>(codes) & 3) || (reinterpret_cast<uintptr_t>(tokens) & 15))
    return fail(FC_ERR_UNSUPPORTED, "codes must be 4-byte and tokens 16-byte aligned");
  int dev = 0, major = 0, nsm = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return fail(FC_ERR_CUDA, std::string("cudaGetDevice: ") + cudaGetErrorString(e));
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (major != 10) return fail(FC_ERR_CUDA, "fc kernels are built for sm_100a only (no CPU/other-arch fallback)");
  static thread_local ExpandParams prm;
  prm.codes = reinterpret_cast<const uint32_t*>(codes);
  prm.tokens = tokens;
  prm.units = static_cast<long long>(rows) * kUnitsPerRow;
  // R5 table (fp32), or its R16 bf16 rounding -- the plan's own normalisation
  for (int i = 0; i < 768; ++i) {
    uint32_t b;
    std::memcpy(&b, &P->lut[i], 4);
    prm.lut[i] = out_dtype == FC_TOKENS_BF16 ? (b + 0x7FFFu + ((b >> 16) & 1u)) >> 16 : b;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const long long want = (prm.units + kThreadsX - 1) / kThreadsX;
  const int grid = static_cast<int>(std::min<long long>(want, static_cast<long long>(nsm) * 8));  // 8 x 256 threads/SM
  if (out_dtype == FC_TOKENS_BF16)
    fc_expand_kernel<FC_TOKENS_BF16><<<grid, kThreadsX, 0, s>>>(prm);
  else
    fc_expand_kernel<FC_TOKENS_F32><<<grid, kThreadsX, 0, s>>>(prm);
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail(FC_ERR_CUDA, std::string("expand launch: ") + cudaGetErrorString(e));
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  return FC_OK;
}
