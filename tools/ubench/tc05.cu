// tc05.cu -- tcgen05 kind::i8 checks on B200 (sm_100a): descriptor layouts
// (K-major / MN-major, no swizzle, arbitrary LBO/SBO), TMEM lane mapping for
// M=64 / M=128, u8 x s8 -> s32 exactness, and per-instruction throughput.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tc05 tc05.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // version 1 (Blackwell)
  return d;                             // base offset 0, lbo mode 0, layout SWIZZLE_NONE
}
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, int amaj, int bmaj, int afmt, int bfmt) {
  return (2u << 4) | (static_cast<uint32_t>(afmt) << 7) | (static_cast<uint32_t>(bfmt) << 10) |
         (static_cast<uint32_t>(amaj) << 15) | (static_cast<uint32_t>(bmaj) << 16) |
         (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t ph) {
  asm volatile(
      "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
          smem_u32(bar)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void ld32x32b_x8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

struct Test {
  int M, N, K;
  int amaj;  // 0 K-major, 1 MN-major
  int lboA, sboA, lboB, sboB;
  int lane_off;  // D lane offset (M=64 interleave test)
};

// A logical [M][K] u8, B logical [N][K] s8; D [M][N] s32
__device__ int offK(int m, int k, int lbo, int sbo) { return (m / 8) * sbo + (k / 16) * lbo + (m % 8) * 16 + (k % 16); }
__device__ int offMN(int m, int k, int lbo, int sbo) { return (m / 16) * sbo + (k / 8) * lbo + (k % 8) * 16 + (m % 16); }

__global__ void k_check(Test t, const uint8_t* A, const int8_t* B, int32_t* D, int abytes) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  uint8_t* sA = sm;
  uint8_t* sB = sm + abytes;
  for (int i = threadIdx.x; i < t.M * t.K; i += blockDim.x) {
    const int m = i / t.K, k = i % t.K;
    sA[t.amaj ? offMN(m, k, t.lboA, t.sboA) : offK(m, k, t.lboA, t.sboA)] = A[i];
  }
  for (int i = threadIdx.x; i < t.N * t.K; i += blockDim.x) {
    const int n = i / t.K, k = i % t.K;
    sB[offK(n, k, t.lboB, t.sboB)] = static_cast<uint8_t>(B[i]);
  }
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  if (threadIdx.x == 0) {
    const uint32_t id = idesc_i8(t.M, t.N, t.amaj, 0, 0, 1);
    for (int kk = 0; kk < t.K / 32; ++kk) {
      const uint32_t aoff = t.amaj ? 4 * kk * t.lboA : 2 * kk * t.lboA;
      const uint64_t a = sdesc(smem_u32(sA) + aoff, t.lboA, t.sboA);
      const uint64_t b = sdesc(smem_u32(sB) + 2 * kk * t.lboB, t.lboB, t.sboB);
      mma_i8(tm + (static_cast<uint32_t>(t.lane_off) << 16), a, b, id, kk > 0);
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp < 4) {
    const int lane = threadIdx.x % 32;
    const int tl = 32 * warp + lane;  // TMEM lane of this thread
    for (int c = 0; c < t.N; c += 8) {
      uint32_t r[8];
      ld32x32b_x8(tm + (static_cast<uint32_t>(32 * warp) << 16) + c, r);
      ld_wait();
      // logical row: M=128 -> lane; M=64 -> lanes (m%16)+32(m/16) (+lane_off)
      int m = -1;
      if (t.M == 128) m = tl;
      else {
        const int q = tl / 32, l = tl % 32 - t.lane_off;
        if (l >= 0 && l < 16) m = 16 * q + l;
      }
      if (m >= 0)
        for (int j = 0; j < 8; ++j) D[m * t.N + c + j] = static_cast<int32_t>(r[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

// throughput: NIT back-to-back MMAs (same operands), cycles per MMA
__global__ void k_tput(int M, int N, int amaj, int nit, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  if (threadIdx.x == 0) {
    const uint32_t id = idesc_i8(M, N, amaj, 0, 0, 1);
    const uint64_t a = sdesc(smem_u32(sm), 128, 1024);
    const uint64_t b = sdesc(smem_u32(sm + 48 * 1024), 128, 1024);
    long long t0 = clock64();
    for (int i = 0; i < nit; ++i) mma_i8(tm + (i & 1) * 256 * 0, a, b, id, 1);
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    cyc[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

static int run_check(const Test& t, unsigned seed) {
  srand(seed);
  std::vector<uint8_t> A(t.M * t.K);
  std::vector<int8_t> B(t.N * t.K);
  for (auto& a : A) a = rand() & 255;
  for (auto& b : B) b = static_cast<int8_t>(rand() & 255);
  std::vector<int32_t> ref(t.M * t.N), got(t.M * t.N, 0x7f7f7f7f);
  for (int m = 0; m < t.M; ++m)
    for (int n = 0; n < t.N; ++n) {
      int s = 0;
      for (int k = 0; k < t.K; ++k) s += static_cast<int>(A[m * t.K + k]) * static_cast<int>(B[n * t.K + k]);
      ref[m * t.N + n] = s;
    }
  uint8_t *dA;
  int8_t* dB;
  int32_t* dD;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dD, got.size() * 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dD, got.data(), got.size() * 4, cudaMemcpyHostToDevice);
  const int abytes = 64 * 1024, smem = 128 * 1024;
  cudaFuncSetAttribute(k_check, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_check<<<1, 256, smem>>>(t, dA, dB, dD, abytes);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(got.data(), dD, got.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (size_t i = 0; i < got.size(); ++i) bad += got[i] != ref[i];
  printf("check M=%d N=%d K=%d %s lboA=%d sboA=%d lboB=%d sboB=%d laneoff=%d: %s, %d/%zu mismatches (got[0]=%d ref[0]=%d, got[last]=%d ref=%d)\n",
         t.M, t.N, t.K, t.amaj ? "A MN-major" : "A K-major", t.lboA, t.sboA, t.lboB, t.sboB, t.lane_off,
         cudaGetErrorString(e), bad, got.size(), got[0], ref[0], got.back(), ref.back());
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  return bad != 0 || e != cudaSuccess;
}

int main() {
  int fails = 0;
  // H-pass style: A K-major (rows x 128 B), B K-major, N = 192
  fails += run_check({128, 192, 128, 0, 128, 1024, 128, 1024, 0}, 1);   // dense core matrices
  fails += run_check({128, 192, 128, 0, 144, 1152, 128, 1024, 0}, 2);   // padded LBO (bank spreading)
  fails += run_check({128, 192, 128, 0, 128, 2048, 3072, 128, 0}, 3);   // B: 8-row groups adjacent, K chunks far apart
  fails += run_check({128, 96, 96, 0, 128, 768, 128, 768, 0}, 4);
  // V-pass style: A MN-major (T rows, x contiguous), B K-major, N = 96
  fails += run_check({128, 96, 96, 1, 128, 1536, 128, 768, 0}, 5);      // LBO = 8-row group stride, SBO = 16-col stride
  fails += run_check({128, 96, 96, 1, 2048, 128, 128, 768, 0}, 6);      // swapped roles
  fails += run_check({128, 256, 64, 1, 128, 1024, 128, 512, 0}, 7);
  // M = 64 (half sub-partitions) with D lane offsets 0 / 16
  fails += run_check({64, 192, 64, 0, 128, 1024, 128, 1024, 0}, 8);
  fails += run_check({64, 192, 64, 0, 128, 1024, 128, 1024, 16}, 9);
  fails += run_check({64, 64, 128, 1, 128, 2048, 128, 1024, 0}, 10);
  printf("check failures: %d\n", fails);

  long long* dc;
  cudaMalloc(&dc, 148 * sizeof(long long));
  cudaFuncSetAttribute(k_tput, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int shapes[][3] = {{128, 256, 0}, {128, 192, 0}, {128, 96, 0}, {128, 64, 0}, {128, 16, 0}, {64, 192, 0},
                           {64, 64, 0},   {128, 96, 1},  {128, 192, 1}};
  for (auto& s : shapes) {
    const int nit = 2048;
    k_tput<<<148, 128, 100 * 1024>>>(s[0], s[1], s[2], nit, dc);
    cudaDeviceSynchronize();
    k_tput<<<148, 128, 100 * 1024>>>(s[0], s[1], s[2], nit, dc);
    cudaError_t e = cudaDeviceSynchronize();
    long long c[148];
    cudaMemcpy(c, dc, sizeof(c), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (long long x : c) mx = x > mx ? x : mx;
    const double per = static_cast<double>(mx) / nit;
    const double macs = static_cast<double>(s[0]) * s[1] * 32;
    printf("tput M=%d N=%d K=32 %s: %.1f clk/MMA, %.0f MAC/clk/SM (%s)\n", s[0], s[1], s[2] ? "A MN" : "A K", per,
           macs / per, cudaGetErrorString(e));
  }
  return fails != 0;
}
