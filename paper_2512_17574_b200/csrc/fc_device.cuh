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

// 2-D tensor copy global -> shared through the TMA engine (UTMALDG): the box
// at element coordinates (x, y) of the tensor map; out-of-bounds bytes are
// zero-filled and still counted in the transaction bytes.
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(tmap), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// Programmatic dependent launch (the launcher sets the attribute): the next
// launch on the stream may start its prologue while this grid drains; its
// threads wait here for every prerequisite grid to complete (and its memory
// to be visible) before touching global data.  No-ops without the attribute.
__device__ __forceinline__ void grid_dependency_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---------------------------------------------------------------- integer math
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
// (sat_u16(a) << 16) | sat_u16(b)
__device__ __forceinline__ uint32_t pack_sat_u16(int a, int b) {
  uint32_t d;
  asm("cvt.pack.sat.u16.s32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
// relu(min(a + b, c)): one VIADDMNMX.RELU
__device__ __forceinline__ int add_min_relu(int a, int b, int c) {
  int d;
  asm("min.relu.s32 %0, %1, %2;" : "=r"(d) : "r"(a + b), "r"(c));
  return d;
}

// Integer YUV -> RGB (R3 BT.601 limited by default; R15 variants) on 4 pixels.  yw = Y0..Y3 bytes, uvw =
// U0 V0 U1 V1 (the chroma samples of pixels {0,1} and {2,3}).  With the
// constants folding C=Y-16, D=U-128, E=V-128 and the +128 rounding:
//   R = (298Y + 409V - 56992) >> 8, G = (298Y - 100U - 208V + 34784) >> 8,
//   B = (298Y + 516U - 70688) >> 8, each saturated to [0,255].
// dp2a forms the two-term dot products straight from byte lanes; the
// saturating pack does the clamp.  Returns one word per channel.
__device__ __forceinline__ void yuv2rgb_4(uint32_t yw, uint32_t uvw, uint32_t& R, uint32_t& G, uint32_t& B,
                                          uint32_t kR, uint32_t kG, uint32_t kGv, uint32_t kB, int bR, int bG,
                                          int bB) {
  // kR = (cRV << 16) | cY, kB = (cBU << 16) | cY, kG = (cGU << 16) | cY, kGv = cGV << 16 (s16 halves)
  // byte words: [Y0 V0 Y1 V0], [Y2 V1 Y3 V1], [Y0 U0 Y1 U0], [Y2 U1 Y3 U1]
  const uint32_t yv01 = __byte_perm(yw, uvw, 0x5150);
  const uint32_t yv23 = __byte_perm(yw, uvw, 0x7372);
  const uint32_t yu01 = __byte_perm(yw, uvw, 0x4140);
  const uint32_t yu23 = __byte_perm(yw, uvw, 0x6362);
  const int g0 = dp2a_lo(kGv, yv01, bG);  // cGV*V0 + bias
  const int g1 = dp2a_lo(kGv, yv23, bG);
  // t -> clamp(t >> 8, 0, 255) == byte 1 of sat_u16(t): pack two saturated
  // halves, then gather the high bytes of four values with one PRMT.
  const uint32_t r01 = pack_sat_u16(dp2a_hi(kR, yv01, bR), dp2a_lo(kR, yv01, bR));
  const uint32_t r23 = pack_sat_u16(dp2a_hi(kR, yv23, bR), dp2a_lo(kR, yv23, bR));
  const uint32_t b01 = pack_sat_u16(dp2a_hi(kB, yu01, bB), dp2a_lo(kB, yu01, bB));
  const uint32_t b23 = pack_sat_u16(dp2a_hi(kB, yu23, bB), dp2a_lo(kB, yu23, bB));
  const uint32_t g01 = pack_sat_u16(dp2a_hi(kG, yu01, g0), dp2a_lo(kG, yu01, g0));
  const uint32_t g23 = pack_sat_u16(dp2a_hi(kG, yu23, g1), dp2a_lo(kG, yu23, g1));
  R = __byte_perm(r01, r23, 0x7531);
  G = __byte_perm(g01, g23, 0x7531);
  B = __byte_perm(b01, b23, 0x7531);
}

// yuv2rgb_4 on two vertically adjacent rows of 4 pixels that share their
// chroma (4:2:0): ye / yo = the even / odd row's Y0..Y3.  The chroma-only
// term of G (cGV*V + bias) is computed once for both rows.
__device__ __forceinline__ void yuv2rgb_4x2(uint32_t ye, uint32_t yo, uint32_t uvw, uint32_t& Re, uint32_t& Ge,
                                            uint32_t& Be, uint32_t& Ro, uint32_t& Go, uint32_t& Bo, uint32_t kR,
                                            uint32_t kG, uint32_t kGv, uint32_t kB, int bR, int bG, int bB) {
  const int g0 = dp2a_lo(kGv, uvw, bG);  // cGV*V0 + bias (kGv's low half is 0: U0 drops out)
  const int g1 = dp2a_hi(kGv, uvw, bG);  // cGV*V1 + bias
  auto row = [&](uint32_t yw, uint32_t& R, uint32_t& G, uint32_t& B) {
    const uint32_t yv01 = __byte_perm(yw, uvw, 0x5150);
    const uint32_t yv23 = __byte_perm(yw, uvw, 0x7372);
    const uint32_t yu01 = __byte_perm(yw, uvw, 0x4140);
    const uint32_t yu23 = __byte_perm(yw, uvw, 0x6362);
    const uint32_t r01 = pack_sat_u16(dp2a_hi(kR, yv01, bR), dp2a_lo(kR, yv01, bR));
    const uint32_t r23 = pack_sat_u16(dp2a_hi(kR, yv23, bR), dp2a_lo(kR, yv23, bR));
    const uint32_t b01 = pack_sat_u16(dp2a_hi(kB, yu01, bB), dp2a_lo(kB, yu01, bB));
    const uint32_t b23 = pack_sat_u16(dp2a_hi(kB, yu23, bB), dp2a_lo(kB, yu23, bB));
    const uint32_t g01 = pack_sat_u16(dp2a_hi(kG, yu01, g0), dp2a_lo(kG, yu01, g0));
    const uint32_t g23 = pack_sat_u16(dp2a_hi(kG, yu23, g1), dp2a_lo(kG, yu23, g1));
    R = __byte_perm(r01, r23, 0x7531);
    G = __byte_perm(g01, g23, 0x7531);
    B = __byte_perm(b01, b23, 0x7531);
  };
  row(ye, Re, Ge, Be);
  row(yo, Ro, Go, Bo);
}

// The same two rows with the chroma terms formed once per chroma pair: c_ch =
// cU*U + cV*V + bias (one dp2a each, shared by the 2x2 pixels of the pair),
// then per pixel and channel one dp2a adding cY*Y -- the Y byte is selected by
// the coefficient pair (cY in the low or the high half), so no byte shuffles.
__device__ __forceinline__ void yuv2rgb_4x2c(uint32_t ye, uint32_t yo, uint32_t uvw, uint32_t& Re, uint32_t& Ge,
                                             uint32_t& Be, uint32_t& Ro, uint32_t& Go, uint32_t& Bo, uint32_t kR,
                                             uint32_t kG, uint32_t kGv, uint32_t kB, int bR, int bG, int bB) {
  const uint32_t kY0 = kR & 0xFFFFu, kY1 = kY0 << 16;                // (cY, 0), (0, cY)
  const uint32_t kRc = kR & 0xFFFF0000u;                              // (0, cRV)  on (U, V)
  const uint32_t kGc = (kG >> 16) | (kGv & 0xFFFF0000u);              // (cGU, cGV)
  const uint32_t kBc = kB >> 16;                                      // (cBU, 0)
  const int r0 = dp2a_lo(kRc, uvw, bR), r1 = dp2a_hi(kRc, uvw, bR);  // chroma pair 0 (pixels 0,1), 1 (2,3)
  const int g0 = dp2a_lo(kGc, uvw, bG), g1 = dp2a_hi(kGc, uvw, bG);
  const int b0 = dp2a_lo(kBc, uvw, bB), b1 = dp2a_hi(kBc, uvw, bB);
  auto row = [&](uint32_t yw, uint32_t& R, uint32_t& G, uint32_t& B) {
    const uint32_t r01 = pack_sat_u16(dp2a_lo(kY1, yw, r0), dp2a_lo(kY0, yw, r0));
    const uint32_t r23 = pack_sat_u16(dp2a_hi(kY1, yw, r1), dp2a_hi(kY0, yw, r1));
    const uint32_t g01 = pack_sat_u16(dp2a_lo(kY1, yw, g0), dp2a_lo(kY0, yw, g0));
    const uint32_t g23 = pack_sat_u16(dp2a_hi(kY1, yw, g1), dp2a_hi(kY0, yw, g1));
    const uint32_t b01 = pack_sat_u16(dp2a_lo(kY1, yw, b0), dp2a_lo(kY0, yw, b0));
    const uint32_t b23 = pack_sat_u16(dp2a_hi(kY1, yw, b1), dp2a_hi(kY0, yw, b1));
    R = __byte_perm(r01, r23, 0x7531);
    G = __byte_perm(g01, g23, 0x7531);
    B = __byte_perm(b01, b23, 0x7531);
  };
  row(ye, Re, Ge, Be);
  row(yo, Ro, Go, Bo);
}

// ---------------------------------------------------------------- int8 MMA
// D = A(16x32 u8, row) * B(32x8, col) + C, s32.  Fragment layout (g = lane/4,
// t = lane%4; verified on B200 by tools/ubench/mma_layout.cu):
//   a0: row g,  k 4t..4t+3   a1: row g+8   a2: k+16   a3: row g+8, k+16
//   b0: col g,  k 4t..4t+3   b1: k+16
//   d0,d1: row g, cols 2t,2t+1   d2,d3: row g+8
template <bool kSignedB>
__device__ __forceinline__ void mma_u8(int (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  if constexpr (kSignedB) {
    asm("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  } else {
    asm("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
}
// Same with a uniform constant accumulator input (d = A*B + c).
template <bool kSignedB>
__device__ __forceinline__ void mma_u8c(int (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1, int c) {
  if constexpr (kSignedB) {
    asm("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%10,%10,%10,%10};"
        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "r"(c));
  } else {
    asm("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%10,%10,%10,%10};"
        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "r"(c));
  }
}

// Exact 22-bit fixed-point FIR as three independent byte-plane MMAs (R4):
//   S = 2^21 + sum px*iw = ((D2 << 8) + D1) << 8) + D0,  D2 = A*B2 + 32,
// D1 = A*B1, D0 = A*B0 (s32, modular == exact).  The planes are independent so
// the three MMAs overlap; the combine is two LEAs on the ALU pipe.
// bf[ks][plane][2]: B fragments of the KS k-steps.
template <int KS>
__device__ __forceinline__ void fir_mma_planes(int (&d2)[4], int (&d1)[4], int (&d0)[4], const uint32_t (&a)[KS][4],
                                               const uint32_t (&bf)[KS][3][2]) {
  // k-step 0 takes its accumulator from constants (32 = Pillow's 2^21
  // rounding term in units of plane 2; 0 for the others), so no register
  // re-initialisation is needed per tile
  mma_u8c<true>(d2, a[0], bf[0][2][0], bf[0][2][1], 32);
  mma_u8c<false>(d1, a[0], bf[0][1][0], bf[0][1][1], 0);
  mma_u8c<false>(d0, a[0], bf[0][0][0], bf[0][0][1], 0);
#pragma unroll
  for (int k = 1; k < KS; ++k) {
    mma_u8<true>(d2, a[k], bf[k][2][0], bf[k][2][1]);
    mma_u8<false>(d1, a[k], bf[k][1][0], bf[k][1][1]);
    mma_u8<false>(d0, a[k], bf[k][0][0], bf[k][0][1]);
  }
}
__device__ __forceinline__ int combine_planes(int d2, int d1, int d0) {
  const uint32_t t = (static_cast<uint32_t>(d2) << 8) + static_cast<uint32_t>(d1);
  return static_cast<int>((t << 8) + static_cast<uint32_t>(d0));
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned s;
  asm volatile("mov.u32 %0, %smid;" : "=r"(s));
  return s;
}
__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void sts16(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"(static_cast<unsigned short>(v)) : "memory");
}

__device__ __forceinline__ uint2 lds64(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}
// the four words of one MMA A fragment (a0..a3 land in consecutive registers)
__device__ __forceinline__ void lds128(uint32_t (&a)[4], uint32_t addr) {
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]) : "r"(addr));
}
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

// predicated streaming stores (no branch) of one token: fp32 bits / bf16 bits
__device__ __forceinline__ void st_cs_pred(float* p, uint32_t v, bool pred) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.cs.b32 [%0], %1;\n}" ::"l"(p), "r"(v),
               "r"(static_cast<int>(pred))
               : "memory");
}
__device__ __forceinline__ void st_cs_pred(uint16_t* p, uint32_t v, bool pred) {
  asm volatile("{\n\t.reg .pred q;\n\t.reg .b16 h;\n\tsetp.ne.b32 q, %2, 0;\n\tcvt.u16.u32 h, %1;\n\t@q st.global.cs.b16 [%0], h;\n}" ::"l"(p),
               "r"(v), "r"(static_cast<int>(pred))
               : "memory");
}

__device__ __forceinline__ void st_cs_pred(uint8_t* p, uint32_t v, bool pred) {
  asm volatile("{\n\t.reg .pred q;\n\t.reg .b16 h;\n\tsetp.ne.b32 q, %2, 0;\n\tcvt.u16.u32 h, %1;\n\t@q st.global.cs.u8 [%0], h;\n}" ::"l"(p),
               "r"(v), "r"(static_cast<int>(pred))
               : "memory");
}

// predicated streaming store of two adjacent tokens (a at p, b at p + 1)
__device__ __forceinline__ void st_cs_pred2(float* p, uint32_t a, uint32_t b, bool pred) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t@q st.global.cs.v2.b32 [%0], {%1, %2};\n}" ::"l"(p),
               "r"(a), "r"(b), "r"(static_cast<int>(pred))
               : "memory");
}
__device__ __forceinline__ void st_cs_pred2(uint16_t* p, uint32_t a, uint32_t b, bool pred) {
  st_cs_pred(reinterpret_cast<float*>(p), __byte_perm(a, b, 0x5410), pred);  // bf16 bits in the low halves
}
__device__ __forceinline__ void st_cs_pred2(uint8_t* p, uint32_t a, uint32_t b, bool pred) {
  st_cs_pred(reinterpret_cast<uint16_t*>(p), __byte_perm(a, b, 0x0040), pred);  // u8 codes in the low bytes
}

}  // namespace fc
