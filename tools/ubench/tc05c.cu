// tc05c.cu -- the V-pass MMA issue pattern of the tcgen05 kernel: units of
// two M128 N48 K32 MMAs (A MN-major), each unit committed to an mbarrier,
// two TMEM accumulator buffers; optionally 8 epilogue warps that wait for the
// unit, tcgen05.ld it and release the buffer (the kernel's V handshake).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tc05c tc05c.cu
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
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t@!p bra W_%=;\n}" ::"r"(
                   smem_u32(bar)), "r"(ph), "r"(0x989680) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// mode 0: MMAs only, no commits; 1: commit per unit, no consumer; 2: full handshake with 8 consumer warps
__global__ void k(int mode, int nunits, int n_per_unit, int N, long long* cyc, uint32_t* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[2], empty[2], done;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
  if (warp == 8) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(smem_u32(&empty[i])));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&done)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  const uint32_t base = smem_u32(sm);
  const uint32_t id = (2u << 4) | (1u << 10) | (1u << 15) | (static_cast<uint32_t>(N >> 3) << 17) | (8u << 24);
  if (warp == 8 && lane == 0) {
    const uint32_t sbo = 9 * 256;
    long long t0 = clock64();
    for (int u = 0; u < nunits; ++u) {
      const int b = u & 1;
      if (mode == 2) wait(&empty[b], ((u >> 1) & 1) ^ 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      for (int kk = 0; kk < n_per_unit; ++kk)
        mma_i8(tm + 384 + b * 64, sdesc(base + 8 * (u % 3) * sbo + ((u * 24 + 32 * kk) % 128) * 16, 128, sbo),
               sdesc(base + 80 * 1024 + kk * 256, 128, 512), id, kk > 0);
      if (mode >= 1) commit(&full[b]);
    }
    commit(&done);
    wait(&done, 0);
    cyc[blockIdx.x] = (clock64() - t0) * 1000 / (static_cast<long long>(nunits) * n_per_unit);
  } else if (warp < 8 && mode == 2) {
    uint32_t acc = 0;
    const uint32_t tl = static_cast<uint32_t>(32 * (warp & 3)) << 16;
    for (int u = 0; u < nunits; ++u) {
      const int b = u & 1;
      wait(&full[b], (u >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      uint32_t r[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(tm + tl + 384 + b * 64 + 8 * (warp >> 2)));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) arrive(&empty[b]);
      for (int i = 0; i < 8; ++i) acc ^= r[i];
    }
    sink[threadIdx.x] = acc;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 8) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
  long long* dc;
  uint32_t* sink;
  cudaMalloc(&dc, 148 * sizeof(long long));
  cudaMalloc(&sink, 512 * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  for (int N : {48, 96})
    for (int npu : {2, 4})
      for (int mode : {0, 1, 2}) {
        k<<<148, 288, 160 * 1024>>>(mode, 3000, npu, N, dc, sink);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[148];
        cudaMemcpy(h, dc, sizeof(h), cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (long long x : h) mx = x > mx ? x : mx;
        printf("N %d, %d MMAs/unit, mode %d (%s): %.1f clk/MMA (%s)\n", N, npu, mode,
               mode == 0 ? "no commits" : mode == 1 ? "commit per unit" : "commit + 8-warp ld handshake", mx / 1000.0,
               cudaGetErrorString(e));
      }
  return 0;
}
