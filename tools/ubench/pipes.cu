// Pipe-throughput microbenchmark for the sm_100a arithmetic choices of the
// fused NV12 -> patch-token kernel. Each kernel runs
// NCH independent accumulation chains per thread so that latency is hidden,
// and reports thread-ops per clock per SM.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define NCH 8
#define ITERS 4096

__global__ void k_ffma_rrr(float* out, float s) {
  float a[NCH], b[NCH], c[NCH];
  for (int i = 0; i < NCH; ++i) { a[i] = threadIdx.x * 0.1f + i; b[i] = s + i; c[i] = 0; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) c[i] = fmaf(a[i], b[i], c[i]);
#pragma unroll
    for (int i = 0; i < NCH; ++i) b[i] = fmaf(a[i], c[i], b[i]);
  }
  float r = 0; for (int i = 0; i < NCH; ++i) r += c[i] + b[i];
  if (r == 1234.5f) out[0] = r;
}
// weight operand warp-uniform (kernel param -> constant bank / uniform reg)
__global__ void k_ffma_uni(float* out, float w0, float w1) {
  float a[NCH], c[NCH];
  for (int i = 0; i < NCH; ++i) { a[i] = threadIdx.x * 0.1f + i; c[i] = 0; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) c[i] = fmaf(a[i], w0, c[i]);
#pragma unroll
    for (int i = 0; i < NCH; ++i) c[i] = fmaf(a[i], w1, c[i]);
  }
  float r = 0; for (int i = 0; i < NCH; ++i) r += c[i];
  if (r == 1234.5f) out[0] = r;
}
__global__ void k_imad_rrr(int* out, int s) {
  int a[NCH], b[NCH], c[NCH];
  for (int i = 0; i < NCH; ++i) { a[i] = threadIdx.x + i; b[i] = s + i; c[i] = 0; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) c[i] = a[i] * b[i] + c[i];
#pragma unroll
    for (int i = 0; i < NCH; ++i) b[i] = a[i] * c[i] + b[i];
  }
  int r = 0; for (int i = 0; i < NCH; ++i) r += c[i] + b[i];
  if (r == 1234567) out[0] = r;
}
__global__ void k_imad_uni(int* out, int w0, int w1) {
  int a[NCH], c[NCH];
  for (int i = 0; i < NCH; ++i) { a[i] = threadIdx.x + i; c[i] = 0; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) c[i] = a[i] * w0 + c[i];
#pragma unroll
    for (int i = 0; i < NCH; ++i) c[i] = a[i] * w1 + c[i];
  }
  int r = 0; for (int i = 0; i < NCH; ++i) r += c[i];
  if (r == 1234567) out[0] = r;
}
__device__ __forceinline__ void ffma2(float2& d, float2 a, float2 b) {
  unsigned long long da = *reinterpret_cast<unsigned long long*>(&a);
  unsigned long long db = *reinterpret_cast<unsigned long long*>(&b);
  unsigned long long dd = *reinterpret_cast<unsigned long long*>(&d);
  asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(dd) : "l"(da), "l"(db));
  d = *reinterpret_cast<float2*>(&dd);
}
__global__ void k_ffma2_uni(float* out, float w0, float w1) {
  float2 a[NCH], c[NCH];
  float2 W0 = make_float2(w0, w0), W1 = make_float2(w1, w1);
  for (int i = 0; i < NCH; ++i) { a[i] = make_float2(threadIdx.x * 0.1f + i, i); c[i] = make_float2(0, 0); }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) ffma2(c[i], a[i], W0);
#pragma unroll
    for (int i = 0; i < NCH; ++i) ffma2(c[i], a[i], W1);
  }
  float r = 0; for (int i = 0; i < NCH; ++i) r += c[i].x + c[i].y;
  if (r == 1234.5f) out[0] = r;
}
__global__ void k_dp4a(int* out, int w0, int w1) {
  int a[NCH], c[NCH];
  for (int i = 0; i < NCH; ++i) { a[i] = threadIdx.x * 0x01010101 + i; c[i] = 0; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) c[i] = __dp4a(a[i], w0, c[i]);
#pragma unroll
    for (int i = 0; i < NCH; ++i) c[i] = __dp4a(a[i], w1, c[i]);
  }
  int r = 0; for (int i = 0; i < NCH; ++i) r += c[i];
  if (r == 1234567) out[0] = r;
}
__global__ void k_dp2a(int* out, int w0, int w1) {
  int a[NCH], c[NCH];
  for (int i = 0; i < NCH; ++i) { a[i] = threadIdx.x * 0x01010101 + i; c[i] = 0; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) c[i] = __dp2a_lo(w0, a[i], c[i]);
#pragma unroll
    for (int i = 0; i < NCH; ++i) c[i] = __dp2a_hi(w1, a[i], c[i]);
  }
  int r = 0; for (int i = 0; i < NCH; ++i) r += c[i];
  if (r == 1234567) out[0] = r;
}
// integer ALU pipe (PRMT / LOP3) alone
__global__ void k_prmt(int* out, int s0, int s1) {
  int a[NCH], c[NCH];
  for (int i = 0; i < NCH; ++i) { a[i] = threadIdx.x + i; c[i] = i * 77; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) c[i] = __byte_perm(c[i], a[i], s0);
#pragma unroll
    for (int i = 0; i < NCH; ++i) c[i] = __byte_perm(c[i], a[i], s1);
  }
  int r = 0; for (int i = 0; i < NCH; ++i) r += c[i];
  if (r == 1234567) out[0] = r;
}
// IMAD (fma pipe) and PRMT (alu pipe) interleaved: do the pipes dual-issue?
__global__ void k_imad_prmt(int* out, int w0, int s0) {
  int a[NCH], c[NCH], d[NCH];
  for (int i = 0; i < NCH; ++i) { a[i] = threadIdx.x + i; c[i] = 0; d[i] = i; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) { c[i] = a[i] * w0 + c[i]; d[i] = __byte_perm(d[i], a[i], s0); }
#pragma unroll
    for (int i = 0; i < NCH; ++i) { c[i] = d[i] * w0 + c[i]; d[i] = __byte_perm(d[i], c[i], s0); }
  }
  int r = 0; for (int i = 0; i < NCH; ++i) r += c[i] + d[i];
  if (r == 1234567) out[0] = r;
}
// FFMA (fma pipe) + IMNMX (alu pipe) interleaved
__global__ void k_ffma_imnmx(float* out, float w0, int lo) {
  float a[NCH], c[NCH]; int d[NCH];
  for (int i = 0; i < NCH; ++i) { a[i] = threadIdx.x * 0.1f + i; c[i] = 0; d[i] = i; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) { c[i] = fmaf(a[i], w0, c[i]); d[i] = max(d[i] + lo, lo * 3); }
#pragma unroll
    for (int i = 0; i < NCH; ++i) { c[i] = fmaf(a[i], w0, c[i]); d[i] = min(d[i], lo * 5 + (int)i); }
  }
  float r = 0; for (int i = 0; i < NCH; ++i) r += c[i] + d[i];
  if (r == 1234.5f) out[0] = r;
}
__global__ void k_i2f(float* out, int s) {
  int a[NCH]; float c[NCH];
  for (int i = 0; i < NCH; ++i) { a[i] = threadIdx.x + i + s; c[i] = 0; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) { c[i] += __uint2float_rn(a[i] & 0xff); a[i] += 3; }
  }
  float r = 0; for (int i = 0; i < NCH; ++i) r += c[i];
  if (r == 1234.5f) out[0] = r;
}
__global__ void k_lds32(int* out, int s) {
  __shared__ int sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i * s;
  __syncthreads();
  int c[NCH];
  for (int i = 0; i < NCH; ++i) c[i] = 0;
  int idx = threadIdx.x & 1023;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) c[i] ^= sm[(idx + i * 32 + (c[i] & 1)) & 4095];
  }
  int r = 0; for (int i = 0; i < NCH; ++i) r += c[i];
  if (r == 1234567) out[0] = r;
}
__global__ void k_lds128(int* out, int s) {
  __shared__ int4 sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = make_int4(i * s, i, i + 1, i + 2);
  __syncthreads();
  int c[NCH];
  for (int i = 0; i < NCH; ++i) c[i] = 0;
  int idx = threadIdx.x & 255;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) { int4 v = sm[(idx + i * 32 + (c[i] & 1)) & 1023]; c[i] ^= v.x + v.y + v.z + v.w; }
  }
  int r = 0; for (int i = 0; i < NCH; ++i) r += c[i];
  if (r == 1234567) out[0] = r;
}
// dynamic shared-memory byte loads (per-lane distinct, conflict-free)
__global__ void k_ldsu8(int* out, int s) {
  __shared__ unsigned char sm[16384];
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) sm[i] = (unsigned char)(i * s);
  __syncthreads();
  int c[NCH];
  for (int i = 0; i < NCH; ++i) c[i] = 0;
  int idx = threadIdx.x * 4;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) c[i] += sm[(idx + i * 128 + (c[i] & 3)) & 16383];
  }
  int r = 0; for (int i = 0; i < NCH; ++i) r += c[i];
  if (r == 1234567) out[0] = r;
}

template <typename F>
void run(const char* name, F launch, double ops_per_thread) {
  int dev; cudaGetDevice(&dev);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int clk_khz; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  const int blocks = sms * 4, threads = 256;
  launch(blocks, threads);  // warm
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) launch(blocks, threads);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ops = ops_per_thread * blocks * threads * 5;
  double per_s = ops / (ms * 1e-3);
  printf("%-14s %8.3f ms  %8.2f Tops/s  %7.1f ops/clk/SM @%d MHz(max)  err=%s\n", name, ms / 5, per_s / 1e12,
         per_s / (sms * (clk_khz * 1e3)), clk_khz / 1000, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  float* fo; int* io; cudaMalloc(&fo, 64); cudaMalloc(&io, 64);
  const double n2 = 2.0 * NCH * ITERS;
  run("ffma_rrr", [&](int b, int t) { k_ffma_rrr<<<b, t>>>(fo, 1.5f); }, n2);
  run("ffma_uni", [&](int b, int t) { k_ffma_uni<<<b, t>>>(fo, 0.25f, -0.5f); }, n2);
  run("ffma2_uni", [&](int b, int t) { k_ffma2_uni<<<b, t>>>(fo, 0.25f, -0.5f); }, 2 * n2);
  run("imad_rrr", [&](int b, int t) { k_imad_rrr<<<b, t>>>(io, 3); }, n2);
  run("imad_uni", [&](int b, int t) { k_imad_uni<<<b, t>>>(io, 3, -5); }, n2);
  run("dp4a(x4)", [&](int b, int t) { k_dp4a<<<b, t>>>(io, 0x01020304, 0x05060708); }, 4 * n2);
  run("dp2a(x2)", [&](int b, int t) { k_dp2a<<<b, t>>>(io, 0x00020003, 0x00050006); }, 2 * n2);
  run("prmt", [&](int b, int t) { k_prmt<<<b, t>>>(io, 0x5410, 0x3276); }, n2);
  run("imad+prmt", [&](int b, int t) { k_imad_prmt<<<b, t>>>(io, 3, 0x5410); }, 2 * n2);
  run("ffma+imnmx", [&](int b, int t) { k_ffma_imnmx<<<b, t>>>(fo, 0.5f, 2); }, 2 * n2);
  run("i2f.u8", [&](int b, int t) { k_i2f<<<b, t>>>(fo, 1); }, 1.0 * NCH * ITERS);
  run("lds32", [&](int b, int t) { k_lds32<<<b, t>>>(io, 3); }, 1.0 * NCH * ITERS);
  run("lds128", [&](int b, int t) { k_lds128<<<b, t>>>(io, 3); }, 1.0 * NCH * ITERS);
  run("ldsu8", [&](int b, int t) { k_ldsu8<<<b, t>>>(io, 3); }, 1.0 * NCH * ITERS);
  return 0;
}
