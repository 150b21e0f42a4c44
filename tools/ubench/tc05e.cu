// tc05e.cu -- issue cost of tcgen05.mma (kind::i8, M128 N192 K32) as the
// surrounding code varies: straight-line (compile-time descriptors), a
// runtime loop run by one thread, a runtime loop run by the whole warp with an
// elected issuer.  Prints cycles per MMA to issue and to complete.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tc05e tc05e.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
               "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
                   smem_u32(bar)), "r"(ph) : "memory");
}
__device__ __forceinline__ bool elect() {
  uint32_t el;
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\tselp.u32 %0, 1, 0, e;\n\t}" : "=r"(el));
  return el != 0;
}
constexpr uint32_t kId = (2u << 4) | (1u << 10) | (24u << 17) | (8u << 24);  // M128 N192 K-major, u8 x s8

__global__ void k(int mode, int nit, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t done;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&done)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  const uint32_t base = smem_u32(sm);
  long long t0 = 0, t1 = 0, t2 = 0;
  if (mode == 0 && threadIdx.x == 0) {  // straight-line: 4 unrolled MMAs per iteration
    t0 = clock64();
    for (int it = 0; it < nit; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        mma_i8(tm + (it & 1) * 192, sdesc(base + (it & 1) * 32768 + kk * 256, 128, 1024),
               sdesc(base + 65536 + kk * 256, 128, 1024), kId, kk > 0);
    }
    t1 = clock64();
    commit(&done);
    wait(&done, 0);
    t2 = clock64();
  } else if (mode == 1 && threadIdx.x == 0) {  // runtime loop, one thread
    t0 = clock64();
    for (int i = 0; i < 4 * nit; ++i) {
      const int it = i >> 2, kk = i & 3;
      mma_i8(tm + (it & 1) * 192, sdesc(base + (it & 1) * 32768 + kk * 256, 128, 1024),
             sdesc(base + 65536 + kk * 256, 128, 1024), kId, kk > 0);
    }
    t1 = clock64();
    commit(&done);
    wait(&done, 0);
    t2 = clock64();
  } else if (mode == 2 && warp == 0) {  // runtime loop, whole warp, elected issuer
    t0 = clock64();
    for (int i = 0; i < 4 * nit; ++i) {
      const int it = i >> 2, kk = i & 3;
      if (elect())
        mma_i8(tm + (it & 1) * 192, sdesc(base + (it & 1) * 32768 + kk * 256, 128, 1024),
               sdesc(base + 65536 + kk * 256, 128, 1024), kId, kk > 0);
      __syncwarp();
    }
    t1 = clock64();
    if (elect()) commit(&done);
    __syncwarp();
    wait(&done, 0);
    t2 = clock64();
  } else if (mode == 3 && threadIdx.x == 0) {  // runtime loop, 4 unrolled MMAs per iteration, runtime D
    t0 = clock64();
    for (int it = 0; it < nit; ++it) {
      const uint32_t d = tm + (it & 1) * 192, a = base + (it & 1) * 32768;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        mma_i8(d, sdesc(a + kk * 256, 128, 1024), sdesc(base + 65536 + kk * 256, 128, 1024), kId, kk > 0);
    }
    t1 = clock64();
    commit(&done);
    wait(&done, 0);
    t2 = clock64();
  }
  if (threadIdx.x == 0) {
    out[2 * blockIdx.x] = (t1 - t0) * 1000 / (4 * nit);
    out[2 * blockIdx.x + 1] = (t2 - t0) * 1000 / (4 * nit);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
  long long* d;
  cudaMalloc(&d, 2 * 148 * sizeof(long long));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  const char* names[] = {"straight-line, 1 thread", "runtime loop, 1 thread", "runtime loop, warp + elect",
                         "loop of 4 unrolled, 1 thread"};
  for (int m = 0; m < 4; ++m) {
    k<<<148, 128, 160 * 1024>>>(m, 1024, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[296];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    long long a = 0, b = 0;
    for (int i = 0; i < 148; ++i) a = h[2 * i] > a ? h[2 * i] : a, b = h[2 * i + 1] > b ? h[2 * i + 1] : b;
    printf("%-30s issue %.1f clk/MMA, complete %.1f clk/MMA (%s)\n", names[m], a / 1000.0, b / 1000.0, cudaGetErrorString(e));
  }
  return 0;
}
