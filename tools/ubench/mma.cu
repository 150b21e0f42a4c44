// Throughput of legacy warp-level integer MMA on sm_100a (mma.sync.m16n8k32
// s8/u8 -> s32), the candidate for the banded resize contractions.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 2048
#define NACC 8
__global__ void k_imma(int* out, int s) {
  unsigned a0 = threadIdx.x * 0x01010101u + s, a1 = a0 ^ 0x5a5a5a5a, a2 = a0 + 3, a3 = a0 * 7;
  unsigned b0 = 0x01020304u + s, b1 = 0x05060708u;
  int acc[NACC][4];
  for (int i = 0; i < NACC; ++i) for (int j = 0; j < 4; ++j) acc[i][j] = 0;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(acc[i][0]), "+r"(acc[i][1]), "+r"(acc[i][2]), "+r"(acc[i][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  int r = 0; for (int i = 0; i < NACC; ++i) for (int j = 0; j < 4; ++j) r += acc[i][j];
  if (r == 1234567) out[0] = r;
}
__global__ void k_hmma(float* out, int s) {
  unsigned a0 = threadIdx.x * 0x3c003c00u + s, a1 = a0, a2 = a0, a3 = a0, b0 = 0x3c003c00u, b1 = b0;
  float acc[NACC][4];
  for (int i = 0; i < NACC; ++i) for (int j = 0; j < 4; ++j) acc[i][j] = 0;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(acc[i][0]), "+f"(acc[i][1]), "+f"(acc[i][2]), "+f"(acc[i][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float r = 0; for (int i = 0; i < NACC; ++i) for (int j = 0; j < 4; ++j) r += acc[i][j];
  if (r == 1234.5f) out[0] = r;
}
int main() {
  int* io; float* fo; cudaMalloc(&io, 64); cudaMalloc(&fo, 64);
  int sms, clk; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0); cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int wpb : {4, 8, 16}) {
    int threads = 32 * wpb, blocks = sms * 2;
    k_imma<<<blocks, threads>>>(io, 1); cudaDeviceSynchronize();
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0); k_imma<<<blocks, threads>>>(io, 1); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double mmas = (double)blocks * wpb * ITERS * NACC;
    printf("imma m16n8k32 u8.s8  warps/SM=%2d: %.3f ms, %.2f mma/clk/SM, %.0f TOPS (int8 MAC=2 ops) err=%s\n", wpb * 2, ms,
           mmas / (ms * 1e-3) / (sms * clk * 1e3), mmas * 4096 * 2 / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    cudaEventRecord(e0); k_hmma<<<blocks, threads>>>(fo, 1); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("hmma m16n8k16 f16    warps/SM=%2d: %.3f ms, %.2f mma/clk/SM, %.0f TFLOPS\n", wpb * 2, ms,
           mmas / (ms * 1e-3) / (sms * clk * 1e3), mmas * 2048 * 2 / (ms * 1e-3) / 1e12);
  }
  return 0;
}
