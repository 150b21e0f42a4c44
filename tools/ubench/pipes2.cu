// Second pipe microbenchmark: saturating pack / relu-min / lea candidates for
// the colour conversion and the resize epilogue.
#include <cstdio>
#include <cuda_runtime.h>
#define NCH 8
#define ITERS 4096
__device__ __forceinline__ unsigned packsat(int a, int b, unsigned c) {
  unsigned d; asm volatile("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d; }
__device__ __forceinline__ int minrelu(int a, int b) {
  int d; asm volatile("min.relu.s32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d; }
__global__ void k_packsat(unsigned* out, int s) {
  int a[NCH]; unsigned c[NCH];
  for (int i = 0; i < NCH; ++i) { a[i] = threadIdx.x * 37 + i - 300; c[i] = i; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) c[i] = packsat(a[i], a[i] + s, c[i]);
  }
  unsigned r = 0; for (int i = 0; i < NCH; ++i) r += c[i]; if (r == 1234567) out[0] = r;
}
__global__ void k_minrelu(int* out, int s) {
  int c[NCH]; for (int i = 0; i < NCH; ++i) c[i] = threadIdx.x * 37 + i - 300;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) c[i] = minrelu(c[i] + s, 65535);
  }
  int r = 0; for (int i = 0; i < NCH; ++i) r += c[i]; if (r == 1234567) out[0] = r;
}
__global__ void k_lea(int* out, int s) {
  int c[NCH], a[NCH]; for (int i = 0; i < NCH; ++i) { c[i] = threadIdx.x * 37 + i; a[i] = i * s; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) c[i] = (a[i] << 8) + c[i];
#pragma unroll
    for (int i = 0; i < NCH; ++i) a[i] = (c[i] << 3) + a[i];
  }
  int r = 0; for (int i = 0; i < NCH; ++i) r += c[i] + a[i]; if (r == 1234567) out[0] = r;
}
__global__ void k_idp_alu_mix(int* out, int w0, int s0) {
  // 2 IDP : 2 ALU (PRMT/SHF) per step -- do fma and alu pipes overlap?
  int a[NCH], c[NCH], d[NCH];
  for (int i = 0; i < NCH; ++i) { a[i] = threadIdx.x * 0x01010101 + i; c[i] = 0; d[i] = i; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) { c[i] = __dp4a(a[i], w0, c[i]); d[i] = __byte_perm(d[i], c[i], s0); }
#pragma unroll
    for (int i = 0; i < NCH; ++i) { c[i] = __dp4a(d[i], w0, c[i]); d[i] = __funnelshift_r(d[i], c[i], s0); }
  }
  int r = 0; for (int i = 0; i < NCH; ++i) r += c[i] + d[i]; if (r == 1234567) out[0] = r;
}
__global__ void k_ffma2_reg(float* out, float s) {
  float2 a[NCH], w[NCH], c[NCH];
  for (int i = 0; i < NCH; ++i) { a[i] = make_float2(threadIdx.x * 0.1f + i, i); w[i] = make_float2(s + i, s - i); c[i] = make_float2(0, 0); }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
      unsigned long long da = *reinterpret_cast<unsigned long long*>(&a[i]), dw = *reinterpret_cast<unsigned long long*>(&w[i]), dc = *reinterpret_cast<unsigned long long*>(&c[i]);
      asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(dc) : "l"(da), "l"(dw));
      c[i] = *reinterpret_cast<float2*>(&dc);
    }
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
      unsigned long long da = *reinterpret_cast<unsigned long long*>(&a[i]), dw = *reinterpret_cast<unsigned long long*>(&w[(i + 1) % NCH]), dc = *reinterpret_cast<unsigned long long*>(&c[i]);
      asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(dc) : "l"(da), "l"(dw));
      c[i] = *reinterpret_cast<float2*>(&dc);
    }
  }
  float r = 0; for (int i = 0; i < NCH; ++i) r += c[i].x + c[i].y; if (r == 1234.5f) out[0] = r;
}
__global__ void k_f2i_sat(unsigned* out, float s) {
  float a[NCH]; unsigned c[NCH];
  for (int i = 0; i < NCH; ++i) { a[i] = threadIdx.x * 0.37f + i * s; c[i] = 0; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) { unsigned v; asm volatile("cvt.rni.sat.u8.f32 %0, %1;" : "=r"(v) : "f"(a[i])); c[i] += v; a[i] += 1.0f; }
  }
  unsigned r = 0; for (int i = 0; i < NCH; ++i) r += c[i]; if (r == 1234567) out[0] = r;
}
template <typename F> void run(const char* name, F launch, double ops) {
  int sms, clk; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0); cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  int b = sms * 4, t = 256; launch(b, t);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) launch(b, t);
  cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ps = ops * b * t * 5 / (ms * 1e-3);
  printf("%-14s %8.3f ms %7.1f ops/clk/SM (%s)\n", name, ms / 5, ps / (sms * clk * 1e3), cudaGetErrorString(cudaGetLastError()));
}
int main() {
  unsigned* uo; int* io; float* fo; cudaMalloc(&uo, 64); cudaMalloc(&io, 64); cudaMalloc(&fo, 64);
  const double n1 = 1.0 * NCH * ITERS;
  run("packsat(I2IP)", [&](int b, int t) { k_packsat<<<b, t>>>(uo, 5); }, n1);
  run("min.relu", [&](int b, int t) { k_minrelu<<<b, t>>>(io, 3); }, n1);
  run("lea", [&](int b, int t) { k_lea<<<b, t>>>(io, 3); }, 2 * n1);
  run("idp+alu", [&](int b, int t) { k_idp_alu_mix<<<b, t>>>(io, 0x01020304, 0x5410); }, 4 * n1);
  run("ffma2_reg(x2)", [&](int b, int t) { k_ffma2_reg<<<b, t>>>(fo, 0.5f); }, 4 * n1);
  run("f2i.rni.sat.u8", [&](int b, int t) { k_f2i_sat<<<b, t>>>(uo, 0.5f); }, n1);
  return 0;
}
