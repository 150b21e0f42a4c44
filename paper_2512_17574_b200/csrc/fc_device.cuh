// fc_device.cuh -- device helpers of the fused kernel: mbarrier / bulk-copy
// (TMA engine) wrappers and the exact integer arithmetic primitives.
#pragma once
#include <cstdint>

namespace fc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "FC_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra FC_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 1-D bulk copy global -> shared through the TMA engine (UBLKCP), completing
// `bytes` of transaction count on `bar`.  16-byte aligned, multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------- integer math
__device__ __forceinline__ uint32_t dp4a_uu(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("dp4a.u32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
// a: four unsigned pixel bytes; b: four signed weight bytes
__device__ __forceinline__ uint32_t dp4a_us(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
// a: two signed 16-bit coefficients; b: pixel bytes 0,1 (lo) or 2,3 (hi)
__device__ __forceinline__ int dp2a_lo(uint32_t a, uint32_t b, int c) {
  int d;
  asm("dp2a.lo.s32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ int dp2a_hi(uint32_t a, uint32_t b, int c) {
  int d;
  asm("dp2a.hi.s32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
// saturating pack: (c << 16) | (sat_u8(a) << 8) | sat_u8(b)
__device__ __forceinline__ uint32_t pack_sat_u8(int a, int b, uint32_t c) {
  uint32_t d;
  asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
// relu(min(a + b, c)): one VIADDMNMX.RELU
__device__ __forceinline__ int add_min_relu(int a, int b, int c) {
  int d;
  asm("min.relu.s32 %0, %1, %2;" : "=r"(d) : "r"(a + b), "r"(c));
  return d;
}

// Exact 22-bit fixed-point FIR over NW words of 4 taps (R4):
//   S = 2^21 + sum px*iw = s0 + 256*s1 + 65536*s2 (int32, modular == exact).
template <int NW>
__device__ __forceinline__ int fir_sum(const uint32_t (&d)[NW], const uint32_t (&w0)[NW], const uint32_t (&w1)[NW],
                                       const uint32_t (&w2)[NW]) {
  uint32_t s0 = 1u << 21, s1 = 0, s2 = 0;
#pragma unroll
  for (int i = 0; i < NW; ++i) {
    s0 = dp4a_uu(d[i], w0[i], s0);
    s1 = dp4a_uu(d[i], w1[i], s1);
    s2 = dp4a_us(d[i], w2[i], s2);
  }
  return static_cast<int>(s0 + (s1 << 8) + (s2 << 16));
}

// Integer BT.601 limited range (R3) on 4 pixels.  yw = Y0..Y3 bytes, uvw =
// U0 V0 U1 V1 (the chroma samples of pixels {0,1} and {2,3}).  With the
// constants folding C=Y-16, D=U-128, E=V-128 and the +128 rounding:
//   R = (298Y + 409V - 56992) >> 8, G = (298Y - 100U - 208V + 34784) >> 8,
//   B = (298Y + 516U - 70688) >> 8, each saturated to [0,255].
// dp2a forms the two-term dot products straight from byte lanes; the
// saturating pack does the clamp.  Returns one word per channel.
__device__ __forceinline__ void bt601_4(uint32_t yw, uint32_t uvw, uint32_t& R, uint32_t& G, uint32_t& B) {
  const uint32_t kR = (409u << 16) | 298u;
  const uint32_t kB = (516u << 16) | 298u;
  const uint32_t kG = ((0x10000u - 100u) << 16) | 298u;   // (298, -100)
  const uint32_t kGv = (0x10000u - 208u) << 16;           // (0, -208)
  // byte words: [Y0 V0 Y1 V0], [Y2 V1 Y3 V1], [Y0 U0 Y1 U0], [Y2 U1 Y3 U1]
  const uint32_t yv01 = __byte_perm(yw, uvw, 0x5150);
  const uint32_t yv23 = __byte_perm(yw, uvw, 0x7372);
  const uint32_t yu01 = __byte_perm(yw, uvw, 0x4140);
  const uint32_t yu23 = __byte_perm(yw, uvw, 0x6362);
  const int g0 = dp2a_lo(kGv, yv01, 34784);  // -208*V0 + 34784
  const int g1 = dp2a_lo(kGv, yv23, 34784);
  const int r0 = dp2a_lo(kR, yv01, -56992) >> 8, r1 = dp2a_hi(kR, yv01, -56992) >> 8;
  const int r2 = dp2a_lo(kR, yv23, -56992) >> 8, r3 = dp2a_hi(kR, yv23, -56992) >> 8;
  const int b0 = dp2a_lo(kB, yu01, -70688) >> 8, b1 = dp2a_hi(kB, yu01, -70688) >> 8;
  const int b2 = dp2a_lo(kB, yu23, -70688) >> 8, b3 = dp2a_hi(kB, yu23, -70688) >> 8;
  const int q0 = dp2a_lo(kG, yu01, g0) >> 8, q1 = dp2a_hi(kG, yu01, g0) >> 8;
  const int q2 = dp2a_lo(kG, yu23, g1) >> 8, q3 = dp2a_hi(kG, yu23, g1) >> 8;
  R = pack_sat_u8(r1, r0, pack_sat_u8(r3, r2, 0));
  G = pack_sat_u8(q1, q0, pack_sat_u8(q3, q2, 0));
  B = pack_sat_u8(b1, b0, pack_sat_u8(b3, b2, 0));
}

__device__ __forceinline__ void st_cs_f2(float* p, float a, float b) {
  asm volatile("st.global.cs.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(a), "f"(b) : "memory");
}

}  // namespace fc
