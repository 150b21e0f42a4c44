// fc_tc.cuh -- the tcgen05 (5th-generation tensor core) version of the fused
// preprocessing kernel: rows a5-a9 of SURVEY.md section 8 in one launch, the
// two exact Pillow-bicubic passes (R4) as kind::i8 MMAs with accumulators in
// tensor memory, warp-specialised roles linked by mbarriers.
//
// What it computes (Alg. 1 l.21-22, P:386-389
// "convert_AVframes_to_tensor_and_resize", and the readings R3-R6 of
// DESIGN.md): for each temporal pair of the sampled NV12 frames,
//   a5  integer BT.601 NV12 -> RGB                                  (R3)
//   a6  horizontal Pillow bicubic, u8 intermediate (clip8)           (R4)
//   a7  vertical Pillow bicubic                                      (R4)
//   a8  rescale + normalise (table)                                  (R5)
//   a9  2x14x14 patchify in 2x2 merge order                          (R6)
// NV12 is read once (TMA boxes), RGB and the H-pass intermediate live in
// shared memory, tokens are written once.
//
// Exactness.  sum px*iw with 22-bit integer weights iw is split over three
// balanced byte digits iw = d2*2^16 + d1*2^8 + d0 (d0, d1 in [-128, 127]), so
// every MMA is u8 x s8 -> s32 and exact; the epilogue recombines
// S = ((D2 << 8) + D1) << 8 + D0 in int32 (modular == exact under Pillow's
// headroom).  Pillow's rounding term 2^21 enters the H pass as a constant
// column (A = 1, plane-2 weight 32) and the V pass through a doubled
// normalisation table indexed by floor(S / 2^21) (floor((S+2^21)/2^22) ==
// floor((floor(S/2^21) + 1) / 2)).
//
// Work unit: one temporal pair x one strip of 56 output columns (2 merge
// blocks), walking down the frame one band (28 output rows) at a time; CTA b
// owns strip b mod nstrips and a contiguous range of (pair, band) items.
// Roles (one CTA per SM, 13 warps):
//   warp 12      TMA: NV12 chunks (16 source rows of both frames), the
//                strip's H weights (once), each band's V weights;
//   warps 8-11   colour: raw NV12 -> RGB rows of the H-pass A operand
//                (K-major core matrices, K-chunk stride 144 B);
//   warp 7       MMA issuer (one thread) + TMEM owner:
//                H: D[128 x 192] (A rows = 6 planes x 16 source rows, N = 3
//                weight digits x 64 outputs), K = KH source columns;
//                V: per band, 3 M-tiles (2 planes x 64 columns) x 2 halves
//                (16 output rows), D[128 x 48], A = the ring (MN-major);
//   warps 4-6    H epilogue: TMEM -> combine, clip8 -> u8 ring rows;
//   warps 0-3    V epilogue: TMEM -> combine, table -> token stores.
// DESIGN.md section 6b.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "fc_device.cuh"
#include "fc_internal.h"

namespace fc {
namespace tc {

// warp roles (24 warps, one CTA per SM).  tcgen05.ld reaches TMEM lane
// quarter (warp % 4) only, so each epilogue role owns whole quarters and two
// warps share a quarter (splitting its columns between them).
// Two layouts (the SM's warp arbiter favours higher warp ids):
//   FC_TC_LAYOUT 0: V epilogue 0..7, H epilogue 8..10 + 12..14, H MMA 11, TMA 15,
//                   colour 16..22, V MMA 23;
//   FC_TC_LAYOUT 1: colour 0..6, TMA 7, V epilogue 8..15, H epilogue 16..18 +
//                   20..22, H MMA 19, V MMA 23 (the busiest roles on top).
#ifndef FC_TC_LAYOUT
#define FC_TC_LAYOUT 1
#endif
constexpr int kVEpiWarps = 8;   // V epilogue: quarter w%4, rows half (w - kVEpi0)/4 of each 16-row unit
constexpr int kHEpiWarps = 6;   // H epilogue: quarters 0..2 (the 96 real A rows), outputs 0..31 (A) / 32..55 (B)
constexpr int kColWarps = 7;
#if FC_TC_LAYOUT == 0
constexpr int kVEpi0 = 0, kHEpiWarpA = 8, kHEpiWarpB = 12, kMmaWarp = 11, kTmaWarp = 15, kColWarp0 = 16;
#else
constexpr int kVEpi0 = 8, kHEpiWarpA = 16, kHEpiWarpB = 20, kMmaWarp = 19, kTmaWarp = 7, kColWarp0 = 0;
#endif
constexpr int kVMmaWarp = 23;   // V-pass MMA issuer (kMmaWarp issues the H pass and owns TMEM)
static_assert(kVEpi0 % 4 == 0 && kHEpiWarpA % 4 == 0 && kHEpiWarpB % 4 == 0, "epilogue warps start at a lane quarter");
__host__ __device__ constexpr bool is_hepi(int w) {
  return (w >= kHEpiWarpA && w < kHEpiWarpA + 3) || (w >= kHEpiWarpB && w < kHEpiWarpB + 3);
}
__host__ __device__ constexpr bool is_col(int w) { return w >= kColWarp0 && w < kColWarp0 + kColWarps; }
constexpr int kWarps = 24;
constexpr int kThreads = 32 * kWarps;
constexpr int kColThreads = 32 * kColWarps;
constexpr int kChunk = 16;        // source rows per chunk
constexpr int kStrip = 56;        // output columns per strip (2 merge blocks)
constexpr int kStripPad = 64;     // MMA columns per strip
constexpr int kNH = 3 * kStripPad;  // H MMA N: 3 weight digits x 64 outputs
constexpr int kNV = 48;             // V MMA N: 3 weight digits x 16 output rows
constexpr int kLboA = 144;          // A_H K-chunk stride (128 + 16: conflict-free colour stores)
constexpr int kNVD = 16;            // V-done barrier slots (bands in flight, host-checked)
constexpr int kMaxBV = 4;           // B_V slots (bands of V weights in flight)
constexpr int kLut2Lo = 97;         // doubled table: index a + 97 for a = floor(S / 2^21) in [-97, 606]
constexpr int kLut2N = 704;
constexpr int kMaxInline = 112;     // frames whose tensor maps travel in the kernel parameters
constexpr int kMaxBands = 128;      // bands whose V window table travels in the kernel parameters
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kHacc = 0;          // H accumulators: columns [0, 384) (2 buffers of 192)
constexpr uint32_t kVacc = 2 * kNH;    // V accumulators: columns [384, 480) (2 buffers of 48)

// mbarrier indices in the barrier block
enum Bar : int {
  kRawFull = 0, kRawEmpty = 4,   // NR <= 4
  kAFull = 8, kAEmpty = 11,      // NA <= 3
  kHFull = 14, kHEmpty = 16,
  kVFull = 18, kVEmpty = 20,
  kBvFull = 22, kBvEmpty = 26,   // NBV <= 4
  kBhFull = 30,
  kVDone = 32,                   // kNVD slots
  kHReady = kVDone + kNVD,       // kNHR slots: chunk cs's ring rows written (H epilogue -> V MMA warp)
  kNumBars = kHReady + 16
};
constexpr int kNHR = 16;  // > NCH + 1 (host-checked): the V warp never lags a full lap of these

// ring position of a pipeline: slot index and the parity of its lap
struct Pipe {
  uint32_t i = 0, ph = 0;
  __device__ __forceinline__ void next(uint32_t n) {
    if (++i == n) {
      i = 0;
      ph ^= 1;
    }
  }
};

struct TcParams {
  int W, H, W2, H2;
  int gh2, gw2, nstrips, npairs, ppj, nframes;
  int KH, KV, BW, NCH, NR, NA, NBV, nchunks;
  int rawb, ahb, bvb;  // bytes per raw stage / A_H stage / B_V slot
  int sbo_a, sbo_v;    // A_H 8-row group stride; ring 16-column group stride
  int off_lut, off_raw, off_ah, off_bh, off_bv, off_ring, off_tab;  // shared-memory offsets (1024-aligned base)
  const int32_t* sx0;    // [nstrips] 16-aligned first source column of each strip
  const uint8_t* hB;     // [nstrips][192 x KH] H weight digits, K-major core matrices
  const uint8_t* vB;     // [gh2][2][48 x KV]  V weight digits per half band
  const int32_t* vys;    // [gh2][2] 8-aligned first source row of each half band's window
  const int32_t* vcl;    // [gh2] last chunk with a nonzero V weight of the band
  const uint32_t* lut2;  // [3][704] token bits, doubled table
  uint32_t ckR, ckG, ckGv, ckB;  // colour matrix (R3/R15), as in fc_fused.cuh
  int cbR, cbG, cbB;
  void* tokens;          // first token row of the launch (fp32)
  void* const* tokj;     // per-job token bases (batch launches) or null
  uint8_t* dbg_src;      // [nframes, H, W, 3] or null
  uint8_t* dbg_rs;       // [nframes, H2, W2, 3] or null
  int frame_base;
  unsigned long long* prof;  // FC_TC_PROF experiments: per warp 8 wait-cycle counters + total, or null
  int ablate;                // FC_TC_ABLATE experiments (PROF instance only): bits skip parts of the work
  const CUtensorMap* tmg;  // device copy of the maps or null -> tm
  // V window starts / last chunks again, in the parameter (constant) bank: the
  // MMA warp indexes them with warp-uniform band numbers, so the descriptors it
  // builds from them stay in uniform registers (no per-MMA R2UR)
  uint16_t cvys[2 * kMaxBands];
  uint16_t cvcl[kMaxBands];
  CUtensorMap tm[2 * kMaxInline];
};

// ---------------------------------------------------------------- tcgen05 PTX
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  // shared-memory matrix descriptor, SWIZZLE_NONE, version 1 (sm_100);
  // layouts verified on B200 by tools/ubench/tc05.cu
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
// instruction descriptor, kind::i8: D s32, A u8, B s8, A K- (0) or MN-major (1), B K-major
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, int amaj) {
  return (2u << 4) | (0u << 7) | (1u << 10) | (static_cast<uint32_t>(amaj) << 15) |
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
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void ldtm16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
// one lane of the (converged) warp: the tcgen05.mma / commit issuer
__device__ __forceinline__ bool elect_one() {
  uint32_t e;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(e));
  return e != 0;
}
// a warp-uniform value the compiler can keep in a uniform register
__device__ __forceinline__ int bcast(int v) { return __shfl_sync(0xffffffffu, v, 0); }
__device__ __forceinline__ void ldtm8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ void sts64(uint32_t addr, uint32_t a, uint32_t b) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(addr), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ void st_cs(float* p, uint32_t v) {
  asm volatile("st.global.cs.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ---------------------------------------------------------------- work walk
// CTA b owns strip b mod nstrips and the contiguous (pair, band) range of its
// group; a "run" is the part of that range inside one pair (the ring restarts).
struct Range {
  int strip, i0, i1;
};
__device__ __forceinline__ Range cta_range(const TcParams& p) {
  const int ns = p.nstrips, q = blockIdx.x / ns;
  Range r;
  r.strip = blockIdx.x - q * ns;
  const int qhi = (gridDim.x + ns - 1) / ns, rr = gridDim.x - (qhi - 1) * ns;
  const int Q = r.strip < rr ? qhi : qhi - 1;
  const long long PB = static_cast<long long>(p.npairs) * p.gh2;
  r.i0 = static_cast<int>(q * PB / Q);
  r.i1 = static_cast<int>((q + 1) * PB / Q);
  return r;
}

// Chunk (source-row block) bounds of a run: chunks kfirst .. klast.
// vys / vcl live in shared memory (copied at kernel start): every role reads
// them in its loop, and an L2 round trip per band sat on the MMA issue path
__device__ __forceinline__ int ld_tab(const int* a) { return *a; }
struct Tabs {
  const int* vys;  // [gh2][2]
  const int* vcl;  // [gh2]
};
__device__ __forceinline__ int run_kfirst(const Tabs& T, int hbA) { return T.vys[2 * hbA] >> 4; }


// Token base of a pair (batch launches: per-job bases).
__device__ __forceinline__ float* pair_tokens(const TcParams& p, int pair) {
  const size_t pair_rows = static_cast<size_t>(p.gh2) * p.gw2 * 4;
  if (p.tokj != nullptr) {
    const int job = pair / p.ppj;
    return static_cast<float*>(p.tokj[job]) + static_cast<size_t>(pair - job * p.ppj) * pair_rows * kCols;
  }
  return static_cast<float*>(p.tokens) + static_cast<size_t>(pair) * pair_rows * kCols;
}

// suspend-hinted wait: the warp sleeps until the phase completes instead of
// spinning through the issue slots the working roles need
__device__ __forceinline__ void wait_bar(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "TC_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra TC_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x989680)
      : "memory");
}

// wait with back-off sleeps: for roles that run ahead of the pipeline (TMA
// refills, colour), where a few hundred ns of wake-up latency is hidden by the
// stage buffers and the issue slots a poll loop burns are not
__device__ __forceinline__ void wait_bar_backoff(uint64_t* bar, uint32_t parity, uint32_t ns) {
  uint32_t done = 0;
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) break;
    __nanosleep(ns);
  }
}

// V epilogue for one (unit half H_, row group VH) of 8 output rows: combine
// the digits, normalise through the doubled table (a8), store each token at
// its patch-order position (a9).  Rows 16H_+8VH+i of the band; compile-time
// row offsets, so every store is [base + immediate].
template <int H_, int VH, bool DBG, int ABL = 0>
__device__ __forceinline__ void vstore(const TcParams& p, const uint32_t (&d0)[8], const uint32_t (&d1)[8],
                                       const uint32_t (&d2)[8], float* base0, float* base1, uint32_t lutc,
                                       uint8_t* dbg) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    constexpr int y0 = 16 * H_ + 8 * VH;
    const int yl = y0 + i;  // output row within the band
    if (yl < 28) {
      const int s = combine_planes(static_cast<int>(d2[i]), static_cast<int>(d1[i]), static_cast<int>(d0[i]));
      const uint32_t v = (ABL & 1) ? static_cast<uint32_t>(s) : lds32(lutc + static_cast<uint32_t>(s >> 21) * 4u);
      if (!(ABL & 32)) st_cs(yl < 14 ? base0 + yl * 14 : base1 + (yl - 14) * 14, v);
      if (DBG && dbg != nullptr) {
        int a = ((s >> 21) + 1) >> 1;  // clip8(floor((S + 2^21) / 2^22))
        a = a < 0 ? 0 : (a > 255 ? 255 : a);
        dbg[static_cast<size_t>(yl) * p.W2 * 3] = static_cast<uint8_t>(a);
      }
    }
  }
}

template <bool DBG, bool PROF = false>
__global__ void __launch_bounds__(kThreads, 1) fc_tc_kernel(const __grid_constant__ TcParams p) {
  // PROF instance: cycles each warp spends in each of its barrier waits (slot k per call site)
  unsigned long long pacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const long long pt0 = PROF ? clock64() : 0;
  auto WB = [&](uint64_t* bar, uint32_t parity, int k, uint32_t ns) {
    if constexpr (PROF) {
      const long long t = clock64();
      wait_bar_backoff(bar, parity, ns);
      pacc[k] += clock64() - t;
    } else {
      wait_bar_backoff(bar, parity, ns);
    }
  };
  auto W = [&](uint64_t* bar, uint32_t parity, int k) {
    if constexpr (PROF) {
      const long long t = clock64();
      wait_bar(bar, parity);
      pacc[k] += clock64() - t;
    } else {
      wait_bar(bar, parity);
    }
  };
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-align the working base (descriptor and TMA destinations)
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kNumBars * 8);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t s_lut = sbase + p.off_lut, s_raw = sbase + p.off_raw, s_ah = sbase + p.off_ah;
  const uint32_t s_bh = sbase + p.off_bh, s_bv = sbase + p.off_bv, s_ring = sbase + p.off_ring;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const Range R = cta_range(p);
  const int X0 = R.strip * kStrip;

  if (tid == 0) {
    for (int i = 0; i < p.NR; ++i) {
      mbar_init(&bars[kRawFull + i], 1);
      mbar_init(&bars[kRawEmpty + i], kColWarps);
    }
    for (int i = 0; i < p.NA; ++i) {
      mbar_init(&bars[kAFull + i], kColWarps);
      mbar_init(&bars[kAEmpty + i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars[kHFull + i], 1);
      mbar_init(&bars[kHEmpty + i], kHEpiWarps);
      mbar_init(&bars[kVFull + i], 1);
      mbar_init(&bars[kVEmpty + i], kVEpiWarps);
    }
    for (int i = 0; i < p.NBV; ++i) {
      mbar_init(&bars[kBvFull + i], 1);
      mbar_init(&bars[kBvEmpty + i], 1);
    }
    mbar_init(&bars[kBhFull], 1);
    for (int i = 0; i < kNVD; ++i) mbar_init(&bars[kVDone + i], 1);
    for (int i = 0; i < kNHR; ++i) mbar_init(&bars[kHReady + i], kHEpiWarps);
    fence_mbar_init();
  }
  if (warp == kMmaWarp) {  // TMEM: 512 columns (one CTA per SM)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = tid; i < 3 * kLut2N; i += kThreads)
    reinterpret_cast<uint32_t*>(smem + p.off_lut)[i] = __ldg(p.lut2 + i);
  int* tab = reinterpret_cast<int*>(smem + p.off_tab);
  for (int i = tid; i < 3 * p.gh2; i += kThreads) tab[i] = i < 2 * p.gh2 ? __ldg(p.vys + i) : __ldg(p.vcl + i - 2 * p.gh2);
  const Tabs T{tab, tab + 2 * p.gh2};
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == kTmaWarp) {
    // ------------------------------------------------------------------ TMA
    if (lane == 0 && R.i0 < R.i1) {
      const CUtensorMap* tm = p.tmg != nullptr ? p.tmg : p.tm;
      const int SX0 = __ldg(p.sx0 + R.strip);
      const uint32_t bhb = static_cast<uint32_t>(kNH * p.KH);
      mbar_arrive_expect_tx(&bars[kBhFull], bhb);
      bulk_g2s(smem + p.off_bh, p.hB + static_cast<size_t>(R.strip) * bhb, bhb, &bars[kBhFull]);
      Pipe rw, bv;  // producer waits on "empty" with the inverted parity: a fresh barrier passes lap 0
      uint32_t jb = 0;  // band sequence number
      for (int i = R.i0; i < R.i1;) {
        const int pair = i / p.gh2, hbA = i - pair * p.gh2, hbB = min(p.gh2, hbA + (R.i1 - i));
        int knext = run_kfirst(T, hbA);
        const CUtensorMap* m0 = &tm[4 * pair];
        for (int hb = hbA; hb < hbB; ++hb, ++jb) {
          // B_V slot reuse: the V MMAs of band jb - NBV are done (its V-done phase)
          if (jb >= static_cast<uint32_t>(p.NBV)) {
            const uint32_t jo = jb - p.NBV;
            W(&bars[kVDone + (jo % kNVD)], (jo / kNVD) & 1, 0);
          }
          mbar_arrive_expect_tx(&bars[kBvFull + bv.i], static_cast<uint32_t>(p.bvb));
          bulk_g2s(smem + p.off_bv + bv.i * p.bvb, p.vB + static_cast<size_t>(hb) * p.bvb, p.bvb, &bars[kBvFull + bv.i]);
          bv.next(p.NBV);
          const int kl = ld_tab(T.vcl + hb);
          for (; knext <= kl; ++knext) {
            WB(&bars[kRawEmpty + rw.i], rw.ph ^ 1, 1, 256);
            uint64_t* fb = &bars[kRawFull + rw.i];
            mbar_arrive_expect_tx(fb, static_cast<uint32_t>(2 * 24 * p.BW));
            uint8_t* dst = smem + p.off_raw + rw.i * p.rawb;
            for (int f = 0; f < 2; ++f) {
              tma_load_2d(dst + f * 24 * p.BW, m0 + 2 * f, SX0, knext * kChunk, fb);
              tma_load_2d(dst + f * 24 * p.BW + 16 * p.BW, m0 + 2 * f + 1, SX0, knext * (kChunk / 2), fb);
            }
            rw.next(p.NR);
          }
        }
        i += hbB - hbA;
      }
    }
  } else if (is_col(warp)) {
    // ------------------------------------------------------------------ colour (a5)
    const int ct = tid - 32 * kColWarp0;
    const int NKC = p.KH >> 4;
    const int items = 2 * kChunk * NKC;  // (frame, row, 16-pixel column group), column group fastest
    const int SX0 = __ldg(p.sx0 + R.strip);
    // this thread's items (KH <= 256: <= 512 items, <= kMaxItems per thread): raw Y / UV offsets, A_H offset
    constexpr int kMaxItems = (2 * kChunk * 16 + kColThreads - 1) / kColThreads;
    int oy[kMaxItems], ouv[kMaxItems], oa[kMaxItems];
    bool last[kMaxItems];
#pragma unroll
    for (int e = 0; e < kMaxItems; ++e) {
      const int it = ct + e * kColThreads;
      const int r = it / NKC, kc = it - r * NKC, f = r >> 4, y = r & 15;
      oy[e] = f * 24 * p.BW + y * p.BW + 16 * kc;
      ouv[e] = f * 24 * p.BW + (16 + (y >> 1)) * p.BW + 16 * kc;
      const int m0 = f * 48 + y;  // A rows (f*3 + c)*16 + y; K-major: (m/8)*SBO + kc*144 + (m%8)*16
      oa[e] = (m0 >> 3) * p.sbo_a + kc * kLboA + (m0 & 7) * 16;
      last[e] = kc == NKC - 1;
    }
    int nmine = 0;
#pragma unroll
    for (int e = 0; e < kMaxItems; ++e) nmine += ct + e * kColThreads < items;
    Pipe rw, ab;
    for (int i = R.i0; i < R.i1;) {
      const int pair = i / p.gh2, hbA = i - pair * p.gh2, hbB = min(p.gh2, hbA + (R.i1 - i));
      const int kf = run_kfirst(T, hbA), kl = ld_tab(T.vcl + hbB - 1);
      for (int k = kf; k <= kl; ++k) {
        WB(&bars[kRawFull + rw.i], rw.ph, 0, 64);
        WB(&bars[kAEmpty + ab.i], ab.ph ^ 1, 1, 64);
        const uint32_t raw = s_raw + rw.i * p.rawb;
        const uint32_t ah = s_ah + ab.i * p.ahb;
#pragma unroll
        for (int e = 0; e < kMaxItems; ++e) {
          if (e >= nmine || (PROF && (p.ablate & 2))) break;
          const uint4 Yv = lds128(raw + oy[e]);
          const uint4 UVv = lds128(raw + ouv[e]);
          uint4 Rv, Gv, Bv;
          yuv2rgb_4(Yv.x, UVv.x, Rv.x, Gv.x, Bv.x, p.ckR, p.ckG, p.ckGv, p.ckB, p.cbR, p.cbG, p.cbB);
          yuv2rgb_4(Yv.y, UVv.y, Rv.y, Gv.y, Bv.y, p.ckR, p.ckG, p.ckGv, p.ckB, p.cbR, p.cbG, p.cbB);
          yuv2rgb_4(Yv.z, UVv.z, Rv.z, Gv.z, Bv.z, p.ckR, p.ckG, p.ckGv, p.ckB, p.cbR, p.cbG, p.cbB);
          yuv2rgb_4(Yv.w, UVv.w, Rv.w, Gv.w, Bv.w, p.ckR, p.ckG, p.ckGv, p.ckB, p.cbR, p.cbG, p.cbB);
          if (DBG && p.dbg_src != nullptr) {
            const int it = ct + e * kColThreads;
            const int r = it / NKC, kc = it - r * NKC, f = r >> 4, y = r & 15;
            const int yy = k * kChunk + y, x = SX0 + 16 * kc;
            if (yy < p.H) {
              const uint32_t cw[3][4] = {{Rv.x, Rv.y, Rv.z, Rv.w}, {Gv.x, Gv.y, Gv.z, Gv.w}, {Bv.x, Bv.y, Bv.z, Bv.w}};
              const size_t fi = static_cast<size_t>(p.frame_base + 2 * pair + f);
              for (int q = 0; q < 16 && x + q < p.W; ++q)
                for (int c = 0; c < 3; ++c)
                  p.dbg_src[((fi * p.H + yy) * p.W + x + q) * 3 + c] = (cw[c][q >> 2] >> (8 * (q & 3))) & 0xFF;
            }
          }
          if (last[e]) {  // the constant column: A = 1 carries Pillow's 2^21 (plane-2 weight 32)
            Rv.w = (Rv.w & 0x00FFFFFFu) | 0x01000000u;
            Gv.w = (Gv.w & 0x00FFFFFFu) | 0x01000000u;
            Bv.w = (Bv.w & 0x00FFFFFFu) | 0x01000000u;
          }
          const uint32_t o0 = ah + oa[e];
          sts128(o0, Rv.x, Rv.y, Rv.z, Rv.w);
          sts128(o0 + 2 * p.sbo_a, Gv.x, Gv.y, Gv.z, Gv.w);  // A row + 16: two 8-row groups further
          sts128(o0 + 4 * p.sbo_a, Bv.x, Bv.y, Bv.z, Bv.w);
        }
        fence_proxy_async();  // generic-proxy stores -> visible to the tensor core
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&bars[kAFull + ab.i]);
          mbar_arrive(&bars[kRawEmpty + rw.i]);
        }
        rw.next(p.NR);
        ab.next(p.NA);
      }
      i += hbB - hbA;
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------------ MMA issuers (a6: warp 11, a7: warp 24)
    // Each issuer warp runs its loop with all lanes (warp-uniform control flow
    // and values, so the descriptors live in uniform registers: per-MMA R2UR
    // moves cost ~200 cycles each, tools/ubench/tc05e.cu) and one elected lane
    // issues.  The H and V streams are independent (the V pass reads the ring
    // the H epilogue writes), so two warps issue them and neither's fixed
    // per-block cost (elect, commit, waits) stalls the other.
    if (R.i0 < R.i1) {
      // the CTA owns all 512 TMEM columns, so the allocation starts at lane 0,
      // column 0: a compile-time accumulator base keeps the MMA operands uniform
      if (tmem != 0) __trap();
      constexpr uint32_t tmem0 = 0;
      constexpr uint32_t idH = idesc_i8(128, kNH, 0);
      const uint32_t sbo_b = static_cast<uint32_t>(p.KH / 16) * 128;
      const int ksh = p.KH >> 5;
      W(&bars[kBhFull], 0, 0);
      tc_fence_after();
      uint32_t cs = 0;
      Pipe ab;
      for (int i = R.i0; i < R.i1;) {
        const int pair = i / p.gh2, hbA = i - pair * p.gh2, hbB = min(p.gh2, hbA + (R.i1 - i));
        const int kf = p.cvys[2 * hbA] >> 4, klast = p.cvcl[hbB - 1];
        for (int k = kf; k <= klast; ++k, ++cs) {
          const uint32_t b = cs & 1;
          W(&bars[kAFull + ab.i], ab.ph, 2);
          if (cs >= 2) W(&bars[kHEmpty + b], ((cs >> 1) & 1) ^ 1, 1);  // the H epilogue drained chunk cs - 2
          tc_fence_after();
          const long long t0 = PROF ? clock64() : 0;
          const uint32_t ah = s_ah + ab.i * p.ahb;
          const uint32_t d = tmem0 + kHacc + b * kNH;
          const int nk = (PROF && (p.ablate & 16)) ? 0 : ksh;
          if (elect_one()) {
            for (int kk = 0; kk < nk; ++kk)
              mma_i8(d, sdesc(ah + kk * 2 * kLboA, kLboA, p.sbo_a), sdesc(s_bh + kk * 256, 128, sbo_b), idH, kk > 0);
            mma_commit(&bars[kHFull + b]);
            mma_commit(&bars[kAEmpty + ab.i]);
          }
          __syncwarp();
          if (PROF) pacc[5] += clock64() - t0;
          ab.next(p.NA);
        }
        i += hbB - hbA;
      }
    }
  } else if (warp == kVMmaWarp) {
    if (R.i0 < R.i1) {
      if (tmem != 0) __trap();
      constexpr uint32_t tmem0 = 0;
      constexpr uint32_t idV = idesc_i8(128, kNV, 1);
      const uint32_t sbo_bv = static_cast<uint32_t>(p.KV / 16) * 128;
      const int ksv = p.KV >> 5;
      uint32_t cs0 = 0, hseen = 0, j = 0;
      int slot0 = 0;  // ring slot of the run's first chunk (cs0 mod NCH)
      Pipe vb, bv;
      for (int i = R.i0; i < R.i1;) {
        const int pair = i / p.gh2, hbA = i - pair * p.gh2, hbB = min(p.gh2, hbA + (R.i1 - i));
        const int kf = p.cvys[2 * hbA] >> 4, klast = p.cvcl[hbB - 1];
        // band tables one band ahead (parameter-bank loads: their latency hides behind the band's MMAs)
        int ys0 = p.cvys[2 * hbA], ys1 = p.cvys[2 * hbA + 1], cl = p.cvcl[hbA];
        for (int hb = hbA; hb < hbB; ++hb, ++j) {
          const int hn = min(hb + 1, p.gh2 - 1);
          const int nys0 = p.cvys[2 * hn], nys1 = p.cvys[2 * hn + 1], ncl = p.cvcl[hn];
          // the band's rows are in the ring: the H epilogue finished its last chunk (and all before)
          const uint32_t c = cs0 + static_cast<uint32_t>(cl - kf);
          while (hseen <= c) {
            W(&bars[kHReady + (hseen % kNHR)], (hseen / kNHR) & 1, 1);
            ++hseen;
          }
          W(&bars[kBvFull + bv.i], bv.ph, 3);
          tc_fence_after();
          const uint32_t bvs = s_bv + bv.i * p.bvb;
          const int nkv = (PROF && (p.ablate & 8)) ? 0 : ksv;
          // ring slot of each half band's first window chunk, and its row offset
          int sl0 = slot0 + ((ys0 >> 4) - kf), sl1 = slot0 + ((ys1 >> 4) - kf);
          while (sl0 >= p.NCH) sl0 -= p.NCH;
          while (sl1 >= p.NCH) sl1 -= p.NCH;
          const uint32_t ab0 = s_ring + (ys0 & 15) * 16, ab1 = s_ring + (ys1 & 15) * 16;
          for (int t = 0; t < 3; ++t)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              W(&bars[kVEmpty + vb.i], vb.ph ^ 1, 4);
              tc_fence_after();
              const long long t0 = PROF ? clock64() : 0;
              const uint32_t abase = (h ? ab1 : ab0) + 8 * t * p.sbo_v;
              const uint32_t d = tmem0 + kVacc + vb.i * kNV;
              const uint32_t bh = bvs + h * kNV * p.KV;
              if (elect_one()) {
                // k-step kk starts 32*kk rows on: two chunks (slots) per step, same offset within the chunk
                int sk = h ? sl1 : sl0;
                for (int kk = 0; kk < nkv; ++kk) {
                  mma_i8(d, sdesc(abase + sk * 256, 128, p.sbo_v), sdesc(bh + kk * 256, 128, sbo_bv), idV, kk > 0);
                  sk += 2;
                  sk -= sk >= p.NCH ? p.NCH : 0;
                }
                mma_commit(&bars[kVFull + vb.i]);
              }
              __syncwarp();
              if (PROF) pacc[6] += clock64() - t0;
              vb.next(2);
            }
          if (elect_one()) mma_commit(&bars[kVDone + (j % kNVD)]);  // ring free (H epilogue) and B_V slot free (TMA)
          __syncwarp();
          bv.next(p.NBV);
          ys0 = nys0;
          ys1 = nys1;
          cl = ncl;
        }
        const int nrun = klast - kf + 1;  // chunks of the run
        cs0 += static_cast<uint32_t>(nrun);
        slot0 += nrun;
        while (slot0 >= p.NCH) slot0 -= p.NCH;
        i += hbB - hbA;
      }
    }
  } else if (is_hepi(warp)) {
    // ------------------------------------------------------------------ H epilogue (a6 -> ring)
    const int q = warp & 3;                      // TMEM lane quarter 0..2
    // this warp's 8-output steps: outputs 0..31 (warps 8..10) / 32..55 (warps 12..14; 56..63 carry no weights)
    const int h0 = warp >= kHEpiWarpB ? 4 : 0, nh = warp >= kHEpiWarpB ? 3 : 4;
    const int m = 32 * q + lane;                 // A row: plane ip = m / 16, source row y = m % 16
    const int ip = m >> 4, y = m & 15;
    const uint32_t tl = static_cast<uint32_t>(32 * q) << 16;
    const uint32_t ringc = s_ring + (ip * 4 + h0 / 2) * p.sbo_v + y * 16;  // + slot * 256
    uint32_t cs = 0, vseen = 0;
    int slot = 0;
    // band iterator for the ring-free condition: band bi, item position within its run
    int bi = R.i0, brun_end = R.i0, bkf = 0, bhb = 0;
    uint32_t bcs0 = 0, bnext_cs0 = 0;
    // sequence number of band bi's first window chunk (past the CTA's last band: never)
    auto band_cfirst = [&]() -> long long {
      if (bi >= R.i1) return 1ll << 40;
      if (bi == brun_end) {  // the iterator enters a new run
        const int bp = bi / p.gh2, bh = bi - bp * p.gh2, be = min(p.gh2, bh + (R.i1 - bi));
        bcs0 = bnext_cs0;
        bkf = run_kfirst(T, bh);
        bhb = bh;
        bnext_cs0 = bcs0 + static_cast<uint32_t>(ld_tab(T.vcl + be - 1) - bkf + 1);
        brun_end = bi + (be - bh);
      }
      return static_cast<long long>(bcs0) + (run_kfirst(T, bhb) - bkf);
    };
    long long ncf = band_cfirst();
    for (int i = R.i0; i < R.i1;) {
      const int pair = i / p.gh2, hbA = i - pair * p.gh2, hbB = min(p.gh2, hbA + (R.i1 - i));
      const int kf = run_kfirst(T, hbA), kl = ld_tab(T.vcl + hbB - 1);
      for (int k = kf; k <= kl; ++k, ++cs) {
        // ring free: chunk cs overwrites chunk cs - NCH, so every band whose
        // window starts at or before chunk cs - NCH must have finished its V MMAs
        while (ncf + p.NCH <= static_cast<long long>(cs)) {
          W(&bars[kVDone + (vseen % kNVD)], (vseen / kNVD) & 1, 0);
          ++vseen;
          ++bi;
          ++bhb;
          ncf = band_cfirst();
        }
        const uint32_t b = cs & 1;
        W(&bars[kHFull + b], (cs >> 1) & 1, 1);
        tc_fence_after();
        // 8-output steps (tcgen05.ld x8 per digit), software-pipelined: the loads
        // of step s+1 are in flight while step s is combined and packed
        const uint32_t taddr = tmem + tl + kHacc + b * kNH + 8 * h0;
        const uint32_t rrow = ringc + slot * 256;
        if (!(PROF && (p.ablate & 4))) {
          uint32_t x0[8], x1[8], x2[8], y0[8], y1[8], y2[8];
          auto load = [&](int st, uint32_t (&e0)[8], uint32_t (&e1)[8], uint32_t (&e2)[8]) {
            ldtm8(taddr + 8 * st, e0);
            ldtm8(taddr + kStripPad + 8 * st, e1);
            ldtm8(taddr + 2 * kStripPad + 8 * st, e2);
          };
          // clip8 (R4) = sat_u8(S >> 22), S = ((D2 << 8) + D1) << 8 + D0; 8 outputs -> 2 words
          // (pack_sat_u8(a, b, c) = c<<16 | sat(a)<<8 | sat(b): bytes [v0 v1 v2 v3])
          auto pack8 = [&](const uint32_t (&e0)[8], const uint32_t (&e1)[8], const uint32_t (&e2)[8], uint32_t& wa,
                           uint32_t& wb) {
            int v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
              v[u] = combine_planes(static_cast<int>(e2[u]), static_cast<int>(e1[u]), static_cast<int>(e0[u])) >> 22;
            wa = pack_sat_u8(v[1], v[0], pack_sat_u8(v[3], v[2], 0u));
            wb = pack_sat_u8(v[5], v[4], pack_sat_u8(v[7], v[6], 0u));
          };
          auto store = [&](uint32_t off, uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3) {
            sts128(off, w0, w1, w2, w3);
            if (slot < 2) sts128(off + p.NCH * 256, w0, w1, w2, w3);  // mirror slot
          };
          uint32_t w0, w1, w2, w3;
          load(0, x0, x1, x2);
          load(1, y0, y1, y2);
          ld_wait();
          pack8(x0, x1, x2, w0, w1);
          pack8(y0, y1, y2, w2, w3);
          if (nh > 2) load(2, x0, x1, x2);
          if (nh > 3) load(3, y0, y1, y2);
          store(rrow, w0, w1, w2, w3);  // outputs 16*(h0/2) .. +15
          if (nh > 2) {
            ld_wait();
            pack8(x0, x1, x2, w0, w1);
            if (nh > 3) {
              pack8(y0, y1, y2, w2, w3);
              store(rrow + p.sbo_v, w0, w1, w2, w3);
            } else {  // outputs 48..55 (56..63 carry no weights: never stored)
              sts64(rrow + p.sbo_v, w0, w1);
              if (slot < 2) sts64(rrow + p.sbo_v + p.NCH * 256, w0, w1);
            }
          }
        }
        fence_proxy_async();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&bars[kHEmpty + b]);            // the H MMA warp may reuse the accumulator
          mbar_arrive(&bars[kHReady + (cs % kNHR)]);  // the V MMA warp may read the ring rows
        }
        if (++slot == p.NCH) slot = 0;
      }
      i += hbB - hbA;
    }
  } else {
    // ------------------------------------------------------------------ V epilogue (a7 -> a8, a9)
    const int q = warp & 3, vh = (warp - kVEpi0) >> 2;  // lane quarter; rows 8vh..8vh+7 of each 16-row unit
    const int m = 32 * q + lane;
    const int pp = m >> 6, x = m & 63;  // plane of the M-tile pair, strip column
    const uint32_t tl = static_cast<uint32_t>(32 * q) << 16;
    const int xvalid = min(kStrip, p.W2 - X0);
    const bool xok = x < xvalid;
    const int wbl = x / 28, wm = (x % 28) / 14, pw = x % 14;
    Pipe vb;
    for (int i = R.i0; i < R.i1;) {
      const int pair = i / p.gh2, hbA = i - pair * p.gh2, hbB = min(p.gh2, hbA + (R.i1 - i));
      float* tpair = pair_tokens(p, pair);
      for (int hb = hbA; hb < hbB; ++hb) {
        // token row of (hm = 0, this column): merge block (hb, X0/28 + wbl), sub-block (0, wm)
        const size_t row0 = (static_cast<size_t>(hb) * p.gw2 + X0 / 28 + wbl) * 4 + wm;
#pragma unroll 1
        for (int t = 0; t < 3; ++t) {
          const int ipl = 2 * t + pp, f = ipl >= 3, c = ipl - 3 * f;
          float* base0 = tpair + row0 * kCols + (c * 2 + f) * 196 + pw;  // hm = 0, ph = 0
          float* base1 = base0 + 2 * kCols;                              // hm = 1
          const uint32_t lutc = s_lut + (c * kLut2N + kLut2Lo) * 4;
          uint8_t* dbg = nullptr;
          if (DBG && p.dbg_rs != nullptr)
            dbg = p.dbg_rs + ((static_cast<size_t>(p.frame_base + 2 * pair + f) * p.H2 + 28 * hb) * p.W2 + X0 + x) * 3 + c;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            W(&bars[kVFull + vb.i], vb.ph, 0);
            tc_fence_after();
            uint32_t d0[8], d1[8], d2[8];
            const uint32_t taddr = tmem + tl + kVacc + vb.i * kNV + 8 * vh;
            ldtm8(taddr, d0);
            ldtm8(taddr + 16, d1);
            ldtm8(taddr + 32, d2);
            ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars[kVEmpty + vb.i]);
            vb.next(2);
            if (PROF && (p.ablate & 33)) {  // ablation experiments: no table (1) / no stores (32)
              if (xok) {
                if (p.ablate & 1) vstore<0, 0, false, 1>(p, d0, d1, d2, base0, base1, lutc, nullptr);
                else vstore<0, 0, false, 32>(p, d0, d1, d2, base0, base1, lutc, nullptr);
              }
            } else if (xok) {
              if (h == 0) {
                if (vh == 0) vstore<0, 0, DBG>(p, d0, d1, d2, base0, base1, lutc, dbg);
                else vstore<0, 1, DBG>(p, d0, d1, d2, base0, base1, lutc, dbg);
              } else {
                if (vh == 0) vstore<1, 0, DBG>(p, d0, d1, d2, base0, base1, lutc, dbg);
                else vstore<1, 1, DBG>(p, d0, d1, d2, base0, base1, lutc, dbg);
              }
            }
          }
        }
      }
      i += hbB - hbA;
    }
  }

  if constexpr (PROF) {
    if (lane == 0 && p.prof != nullptr) {
      unsigned long long* o = p.prof + (static_cast<size_t>(blockIdx.x) * kWarps + warp) * 9;
      for (int k = 0; k < 8; ++k) o[k] = pacc[k];
      o[8] = clock64() - pt0;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kMmaWarp)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
}

using TcKernelFn = void (*)(TcParams);
void tc_kernels(TcKernelFn* prod, TcKernelFn* dbg, TcKernelFn* prof);  // fc_tc.cu

}  // namespace tc
}  // namespace fc
