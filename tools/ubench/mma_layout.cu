// Verifies the m16n8k32 u8 x s8 -> s32 fragment layout assumed by the resize
// kernel: A row-major 16x32 (a0: row g, k 4t..4t+3; a1: row g+8; a2: k+16;
// a3: row g+8, k+16), B col-major 32x8 (b0: col g, k 4t..; b1: k+16),
// D (d0,d1: row g, cols 2t,2t+1; d2,d3: row g+8).  g = lane/4, t = lane%4.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k(const uint8_t* A, const int8_t* B, int* D) {
  int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  auto ld = [&](const uint8_t* p) { return (unsigned)p[0] | ((unsigned)p[1] << 8) | ((unsigned)p[2] << 16) | ((unsigned)p[3] << 24); };
  unsigned a0 = ld(A + g * 32 + 4 * t), a1 = ld(A + (g + 8) * 32 + 4 * t), a2 = ld(A + g * 32 + 16 + 4 * t), a3 = ld(A + (g + 8) * 32 + 16 + 4 * t);
  unsigned b0 = ld((const uint8_t*)B + g * 32 + 4 * t), b1 = ld((const uint8_t*)B + g * 32 + 16 + 4 * t);  // B stored as [n][k]
  int d0 = 7, d1 = 7, d2 = 7, d3 = 7;
  asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+r"(d0), "+r"(d1), "+r"(d2), "+r"(d3) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  D[g * 8 + 2 * t] = d0; D[g * 8 + 2 * t + 1] = d1; D[(g + 8) * 8 + 2 * t] = d2; D[(g + 8) * 8 + 2 * t + 1] = d3;
}
int main() {
  uint8_t hA[16 * 32]; int8_t hB[8 * 32]; int hD[128], ref[128];
  for (int i = 0; i < 512; ++i) hA[i] = (uint8_t)(i * 37 + 11);
  for (int i = 0; i < 256; ++i) hB[i] = (int8_t)(i * 53 - 100);
  for (int m = 0; m < 16; ++m) for (int n = 0; n < 8; ++n) { int s = 7; for (int kk = 0; kk < 32; ++kk) s += hA[m * 32 + kk] * hB[n * 32 + kk]; ref[m * 8 + n] = s; }
  uint8_t* dA; int8_t* dB; int* dD; cudaMalloc(&dA, 512); cudaMalloc(&dB, 256); cudaMalloc(&dD, 512);
  cudaMemcpy(dA, hA, 512, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(dA, dB, dD); cudaMemcpy(hD, dD, 512, cudaMemcpyDeviceToHost);
  int bad = 0; for (int i = 0; i < 128; ++i) bad += hD[i] != ref[i];
  printf("mma m16n8k32 layout check: %d mismatches of 128 (%s)\n", bad, cudaGetErrorString(cudaGetLastError()));
  // cvt.pack.sat.u16.s32 semantics probe
  return bad != 0;
}
