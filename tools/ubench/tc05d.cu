// tc05d.cu -- what a switch of the accumulator (D) address costs between
// kind::i8 MMAs on B200: runs of R MMAs into one D, alternating between two
// D column offsets, for several N / A layouts.  No commits inside the loop.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tc05d tc05d.cu
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

__global__ void k(int N, int amaj, int run, int d0, int d1, int accmode, int nmma, int warpmode, long long* cyc) {
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
  const uint32_t id = (2u << 4) | (1u << 10) | (static_cast<uint32_t>(amaj) << 15) | (static_cast<uint32_t>(N >> 3) << 17) |
                      (8u << 24);
  if ((warpmode == 0 && threadIdx.x == 0) || (warpmode == 1 && warp == 0)) {
    // warpmode 0: one thread runs the loop (the kernel's MMA role today);
    // warpmode 1: the whole warp runs it, one elected lane issues each MMA
    long long t0 = clock64();
    for (int i = 0; i < nmma; ++i) {
      const int r = i / run, kk = i % run;
      const uint32_t d = tm + ((r & 1) ? d1 : d0);
      const uint32_t acc = accmode == 0 ? (kk > 0) : accmode == 1 ? 1u : 0u;
      const uint64_t a = amaj ? sdesc(base + ((i * 24) % 128) * 16, 128, 2304) : sdesc(base + (i % 4) * 256, 128, 1024);
      if (warpmode == 0) {
        mma_i8(d, a, sdesc(base + 96 * 1024 + (i % 4) * 256, 128, 1024), id, acc);
      } else {
        uint32_t el;
        asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\tselp.u32 %0, 1, 0, e;\n\t}" : "=r"(el));
        if (el) mma_i8(d, a, sdesc(base + 96 * 1024 + (i % 4) * 256, 128, 1024), id, acc);
        __syncwarp();
      }
    }
    if (threadIdx.x == 0) commit(&done);
    wait(&done, 0);
    if (threadIdx.x == 0) cyc[blockIdx.x] = (clock64() - t0) * 1000 / nmma;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
  long long* dc;
  cudaMalloc(&dc, 148 * sizeof(long long));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  struct C { int N, amaj, run, d0, d1, acc; } cs[] = {
      {48, 1, 1000000, 384, 384, 0}, {48, 1, 6, 384, 432, 0}, {48, 1, 2, 384, 432, 0}, {48, 1, 2, 384, 448, 0},
      {48, 1, 2, 384, 384, 0},       {48, 1, 2, 384, 432, 1}, {48, 1, 1, 384, 432, 2}, {48, 1, 1, 384, 432, 1},
      {48, 0, 2, 384, 432, 0},       {192, 0, 4, 0, 192, 0},  {192, 0, 1000000, 0, 0, 0}, {192, 0, 4, 0, 0, 0},
      {192, 0, 4, 0, 192, 1},        {192, 0, 1, 0, 192, 2},  {96, 1, 2, 384, 0, 0}};
  for (int wm = 0; wm < 2; ++wm)
  for (auto& c : cs) {
    k<<<148, 128, 160 * 1024>>>(c.N, c.amaj, c.run, c.d0, c.d1, c.acc, 4096, wm, dc);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, dc, sizeof(h), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (long long x : h) mx = x > mx ? x : mx;
    printf("%s N %3d A %s run %7d D %3d/%3d acc %s: %.1f clk/MMA (%s)\n", wm ? "warp+elect" : "1 thread  ", c.N, c.amaj ? "MN" : "K ", c.run, c.d0, c.d1,
           c.acc == 0 ? "first-of-run-off" : c.acc == 1 ? "always-on" : "always-off", mx / 1000.0, cudaGetErrorString(e));
  }
  return 0;
}
