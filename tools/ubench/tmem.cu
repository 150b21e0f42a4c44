// tmem.cu -- TMEM read (tcgen05.ld) throughput on B200 per SM, alone and while
// one thread issues kind::i8 MMAs (M128 N192) into other TMEM columns.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tmem tmem.cu
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
template <int X>
__device__ __forceinline__ uint32_t ld(uint32_t taddr) {
  uint32_t r[X];
  if constexpr (X == 16)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
                   "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(taddr));
  else
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  uint32_t s = 0;
  for (int i = 0; i < X; ++i) s ^= r[i];
  return s;
}

// nw reader warps (warp w reads lane quarter w%4, columns [0,192)), optional MMA thread in warp nw
template <int X>
__global__ void k(int nw, int mma, int nit, long long* out, uint32_t* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tbase;
  __shared__ int done;
  __shared__ unsigned long long mcount;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) { done = 0; mcount = 0; }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  if (warp < nw) {
    const uint32_t ta = tm + (static_cast<uint32_t>(32 * (warp & 3)) << 16);
    uint32_t s = 0;
    long long t0 = clock64();
    for (int it = 0; it < nit; ++it)
      for (int c = 0; c < 192; c += X) s ^= ld<X>(ta + c);
    long long t1 = clock64();
    if (lane == 0) out[blockIdx.x * 64 + warp] = t1 - t0;
    sink[threadIdx.x] = s;
    __syncwarp();
    if (lane == 0) atomicAdd(&done, 1);
  } else {
    if (mma && lane == 0 && warp == nw) {
      const uint32_t base = smem_u32(sm);
      unsigned long long n = 0;
      while (atomicAdd(&done, 0) < nw) {
        for (int kk = 0; kk < 4; ++kk, ++n)
          mma_i8(tm + 256, sdesc(base + kk * 256, 128, 1024), sdesc(base + 65536 + kk * 256, 128, 1024),
                 (2u << 4) | (1u << 10) | (24u << 17) | (8u << 24), 1);
      }
      mcount = n;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x * 64 + 63] = mcount;
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
  long long* d;
  uint32_t* sink;
  cudaMalloc(&d, 148 * 64 * sizeof(long long));
  cudaMalloc(&sink, 2048 * 4);
  const int nit = 2000;
  for (int x : {8, 16})
    for (int nw : {1, 4, 8, 16})
      for (int mma : {0, 1}) {
        auto fn = x == 8 ? k<8> : k<16>;
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
        const int threads = 32 * (nw + 1);
        fn<<<148, threads, 150 * 1024>>>(nw, mma, nit, d, sink);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[64];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int w = 0; w < nw; ++w) mx = h[w] > mx ? h[w] : mx;
        const double bytes = static_cast<double>(nw) * nit * 192 * 32 * 4;
        printf("x%-2d readers %2d mma %d: %.1f B/clk/SM (%.0f clk), %lld MMAs meanwhile (%s)\n", x, nw, mma, bytes / mx,
               static_cast<double>(mx), h[63], cudaGetErrorString(e));
      }
  return 0;
}
