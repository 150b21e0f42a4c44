// tc05b.cu -- throughput of the tcgen05 kernel's exact MMA sequences on B200:
// H pass (M128 N192, K=128 in 4 k-steps, A K-major with K-chunk stride LBO
// 128 / 144) and V pass (M128 N48, K=64 in 2 k-steps, A MN-major), each
// k-step reading a different A / B slice, optionally with 8 other warps
// streaming shared memory (LDS.128 + STS.128) at the same time.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tc05b tc05b.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, int amaj) {
  return (2u << 4) | (1u << 10) | (static_cast<uint32_t>(amaj) << 15) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
               "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
                   smem_u32(bar)), "r"(ph) : "memory");
}

// mode 0: H sequence (lboA), mode 1: V sequence; noise: other warps stream smem
__global__ void k(int mode, int lboA, int noise, int nit, long long* cyc, int* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ volatile int stop;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    stop = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  const uint32_t base = smem_u32(sm);
  if (threadIdx.x == 0) {
    long long t0 = clock64();
    int n = 0;
    for (int it = 0; it < nit; ++it) {
      if (mode == 0) {  // H: A [128 rows][128 K] at base (sbo = 8 * lboA), B [192][128] at base + 64K
        const uint32_t sbo = 8 * lboA;
        for (int kk = 0; kk < 4; ++kk, ++n)
          mma_i8(tm + (it & 1) * 192, sdesc(base + (it & 1) * 32768 + kk * 2 * lboA, lboA, sbo),
                 sdesc(base + 65536 + kk * 256, 128, 1024), idesc_i8(128, 192, 0), kk > 0);
      } else {  // V: A MN-major ring, 24 16-column groups x 160 rows; B [48][64]
        const uint32_t sbo = 160 * 16;
        for (int t = 0; t < 3; ++t)
          for (int kk = 0; kk < 2; ++kk, ++n)
            mma_i8(tm + 384 + (it & 1) * 48, sdesc(base + 8 * t * sbo + ((it * 24 + 32 * kk) % 128) * 16, 128, sbo),
                   sdesc(base + 90000 / 1024 * 1024 + kk * 256, 128, 512), idesc_i8(128, 48, 1), kk > 0);
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    cyc[blockIdx.x] = (t1 - t0) * 1000 / n;  // milli-cycles per MMA
    stop = 1;
  } else if (noise && warp >= 1) {  // stream shared memory: 16 B per lane loads + stores
    uint32_t acc = 0;
    const uint32_t off = 120 * 1024 + (threadIdx.x * 16) % 65536;
    while (!stop) {
      for (int r = 0; r < 64; ++r) {
        uint4 v;
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(base + off));
        acc += v.x ^ v.w;
        asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(base + ((off + 4096) & 0x1FFFF) + 120 * 1024 - 120 * 1024), "r"(acc), "r"(v.y), "r"(v.z), "r"(acc) : "memory");
      }
    }
    sink[threadIdx.x] = acc;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
  long long* dc;
  int* sink;
  cudaMalloc(&dc, 148 * sizeof(long long));
  cudaMalloc(&sink, 1024 * sizeof(int));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct C { int mode, lbo, noise; const char* name; } cs[] = {
      {0, 128, 0, "H N192 LBO128"}, {0, 144, 0, "H N192 LBO144"}, {1, 128, 0, "V N48 MN-major"},
      {0, 128, 1, "H N192 LBO128 + smem noise"}, {0, 144, 1, "H N192 LBO144 + smem noise"}, {1, 128, 1, "V N48 + smem noise"}};
  for (auto& c : cs) {
    for (int rep = 0; rep < 2; ++rep) k<<<148, 288, 200 * 1024>>>(c.mode, c.lbo, c.noise, 512, dc, sink);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, dc, sizeof(h), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (long long x : h) mx = x > mx ? x : mx;
    printf("%-30s %.1f clk/MMA (%s)\n", c.name, mx / 1000.0, cudaGetErrorString(e));
  }
  return 0;
}
