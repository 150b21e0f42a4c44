// fc_kernels.cu -- the fused sm_100a kernel of the preprocessing hot path and
// its launcher (fc_preprocess / fc_preprocess_debug / fc_preprocess_batch).
//
// One launch per rank computes, for each temporal pair of the rank's sampled
// frames (Alg. 1 l.21-22, "convert_AVframes_to_tensor_
// and_resize"):
//   a5  NV12 -> RGB, integer BT.601 limited range            (R3)
//   a6  horizontal Pillow-bicubic pass, u8 intermediate      (R4)
//   a7  vertical Pillow-bicubic pass                          (R4)
//   a8  rescale + normalise through a 3x256 fp32 table        (R5)
//   a9  temporal pad + 14x14x2 patchify in 2x2 merge order    (R6)
// in ONE pass over HBM: NV12 bytes are read once (plus strip halos), tokens
// are written once.  See DESIGN.md "Kernel" for the work decomposition and
// its roofline.
//
// Work unit (CTA): one temporal pair x one strip of K merge-block columns
// (SW = 28K output columns), walking down the frame one merge-block row
// (28 output rows, a "band") at a time.  Source rows are converted and
// horizontally filtered once each into a ring of u8 rows (column-major, so
// that 4 vertically adjacent taps are one 32-bit word); the vertical pass
// reads the ring.  All resize MACs are exact integer DP4A on byte planes of
// Pillow's 22-bit weights:  sum px*iw = d0 + 256*d1 + 65536*d2.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <atomic>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <type_traits>
#include <unordered_map>
#include <vector>

#include "fc_device.cuh"
#include "fc_internal.h"

namespace fc {

constexpr int kChunkRows = 16;             // source rows per chunk
constexpr int kTileN = 8;                  // outputs per H-pass MMA tile (N of m16n8k32)
constexpr int kStrip = 56;                 // output columns per strip: 2 merge blocks = 4 patches
constexpr int kComputeWarps = 8;
constexpr int kPlanesPerWarp = 24 / kComputeWarps;  // V pass: (4 row groups x 6 planes) / warps
static_assert(kPlanesPerWarp == 3, "V pass: each warp owns the 3 channels of one frame");
constexpr int kComputeThreads = 32 * kComputeWarps;
constexpr int kThreads = kComputeThreads;  // thread 0 also issues the TMA copies
constexpr int kMaxInlineFrames = 120;      // tensor maps (2 per frame) passed by value up to this many frames
constexpr int kRingStride = 6 * kStrip + 24;  // ring row stride (words): == 8 mod 32, conflict-free A loads
static_assert(kRingStride % 32 == 8, "ring stride must be 8 mod 32");
constexpr int kStages = 4;                 // raw NV12 chunk buffers (TMA runs kStages-1 chunks ahead)
constexpr int kIssueWarp = kComputeWarps - 1;  // owns no H-pass tile (7 tiles of 8 cover a 56-column strip)
static_assert((kStrip + kTileN - 1) / kTileN < kComputeWarps, "the TMA issuing warp must own no H tile");

struct Params {
  int W, H, W2, H2;
  int gh2, gw2;       // merge blocks per column / row
  int nstrips, npairs;
  int sw, htiles;      // strip width (84 or 28 output columns), H tiles per strip
  int SWP;            // RGB-plane row stride (odd multiple of 16)
  int SWPN;           // converted (and TMA-loaded) bytes per row: taps of the strip's outputs
  int BW, NX;         // TMA box width (<= 256) and boxes per row: NX*BW >= SWPN
  int bwshift, bwmask;  // box index / offset of a byte column (NX == 1: 31 / ~0; else BW = 256: 8 / 255)
  int TR, TRW;        // ring rows / words
  int nchunks;        // chunks any band needs
  const int32_t* hx;    // H table: xmin per output column
  const int32_t* hxs;   // H MMA tiles: 4-aligned window start per tile of 8 outputs
  const uint32_t* hfr;  // H MMA tiles: B fragments [tile][KS][3][32][2]
  const int32_t* vx;    // V table: ymin / count per output row
  const int32_t* vcnt;
  const int32_t* vys;   // V MMA groups: 4-aligned window start per (band, group of 8 rows)
  const uint32_t* vfr;  // V MMA groups: B fragments [group][KS][3][32][2]
  const uint32_t* lut;  // 3 x 256 token bits (fp32, or bf16 zero-extended)
  uint32_t ckR, ckG, ckGv, ckB;  // colour matrix (R3/R15): packed s16 (Y, chroma) coefficient pairs for dp2a
  int cbR, cbG, cbB;             // colour biases: -y0*cY - 128*(chroma coefficients) + 128
  void* tokens;       // first token row of this launch's first pair
  uint8_t* dbg_src;   // [nframes_total, H, W, 3] or null
  uint8_t* dbg_rs;    // [nframes_total, H2, W2, 3] or null
  int frame_base;     // index of fr[0] within the rank's frame list (debug dumps)
  uint32_t trw_magic;  // ceil(2^32 / TRW): x mod TRW = x - TRW * umulhi(x, magic) for the row words used
  int nframes;
  int ppj;            // pairs per job (batch launches; == npairs for one job)
  void* const* tokj;  // device: per-job token base (batch launches) or null -> tokens
  const CUtensorMap* tmg;  // device copy of the maps (launches past kMaxInlineFrames frames) or null -> tm
  CUtensorMap tm[2 * kMaxInlineFrames];  // per frame: Y plane (box BW x 16), UV plane (box BW x 8)
};

// Walk of one CTA's work: contiguous (pair, strip, band) items, split into
// runs that stay inside one (pair, strip).
struct Run {
  int pair, strip, hb0, hb1, kfirst, klast;
};

__device__ __forceinline__ bool next_run(const Params& p, int& cur, int i1, Run& r) {
  if (cur >= i1) return false;
  const int ps = cur / p.gh2;
  r.hb0 = cur - ps * p.gh2;
  r.pair = ps / p.nstrips;
  r.strip = ps - r.pair * p.nstrips;
  r.hb1 = min(p.gh2, r.hb0 + (i1 - cur));
  cur += r.hb1 - r.hb0;
  r.kfirst = (__ldg(p.vx + 28 * r.hb0) & ~3) / kChunkRows;
  r.klast = min(p.nchunks, (__ldg(p.vx + 28 * r.hb1 - 1) + __ldg(p.vcnt + 28 * r.hb1 - 1) + kChunkRows - 1) / kChunkRows);
  return true;
}

// Issue the TMA tensor copies of one 16-row chunk into a raw stage (one
// thread): per frame of the pair, NX boxes of Y (BW x 16 rows) then NX boxes
// of UV (BW x 8 rows), after arming the stage's full barrier with their bytes.
__device__ __forceinline__ void issue_chunk(const Params& p, int pair, int SX0, int k, uint8_t* raw, uint64_t* bar) {
  const CUtensorMap* tm = p.tmg != nullptr ? p.tmg : p.tm;
  fence_proxy_async();
  mbar_arrive_expect_tx(bar, static_cast<uint32_t>(2 * 24 * p.BW * p.NX));
  for (int f = 0; f < 2; ++f)
    for (int pl = 0; pl < 2; ++pl)
      for (int sub = 0; sub < p.NX; ++sub) {
        uint8_t* dst = raw + f * 24 * p.BW * p.NX + (pl ? 16 * p.BW * p.NX + sub * 8 * p.BW : sub * 16 * p.BW);
        tma_load_2d(dst, &tm[2 * (2 * pair + f) + pl], SX0 + sub * p.BW,
                    pl ? k * (kChunkRows / 2) : k * kChunkRows, bar);
      }
}

// Persistent, warp-specialised fused kernel.
//   warp 12      : TMA producer -- streams NV12 rows of the next chunk into a
//                  double-buffered raw area (full/empty mbarriers).
//   warps 0..11  : a5 colour (integer BT.601, dp2a) -> RGB planes;
//                  a6 horizontal pass: warp w < 11 owns output tile w (8 columns)
//                  of the strip; three chained int8 MMAs per 16 rows x 8 outputs
//                  -> u8 ring (4 source rows per 32-bit word);
//                  a7 vertical pass: warp w owns 8-row group (w&3) of the band and
//                  planes {2(w>>2), 2(w>>2)+1}; one MMA tile per 14-column patch,
//                  then a8 table + a9 patch-order stores.
// Work items are (pair, strip, band) triples; CTA b takes [b*T/G, (b+1)*T/G).
// Strips are whole merge blocks, so every token row is written by one CTA in
// one band (no partial-sector merging across CTAs in L2).
template <int KSH, int KSV, bool DBG, int TOK>
__global__ void __launch_bounds__(kThreads, 3) fc_fused_kernel(const __grid_constant__ Params p) {
  constexpr int SW = kStrip;
  constexpr int CH = kChunkRows;
  constexpr int RS = kRingStride;

  extern __shared__ __align__(1024) uint8_t smem[];
  uint32_t* lut = reinterpret_cast<uint32_t*>(smem);              // 3 x 256 token bits at offset 0
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + 3072);      // kStages full barriers
  const int RAWF = 24 * p.BW * p.NX;                              // raw bytes per frame per stage
  uint8_t* raw = smem + 3072 + 128;                               // [kStages][2 f][Y boxes | UV boxes]
  const int SWP = p.SWP;
  uint8_t* rgb = raw + kStages * 2 * RAWF;                        // [2 f][3 c][16 rows][SWP]
  uint32_t* ring = reinterpret_cast<uint32_t*>(rgb + 6 * CH * SWP);  // [TRW][RS] words: [w][f][c][x]

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tq = lane & 3;
  const bool issuer = tid == kIssueWarp * 32;  // lane 0 of the warp without an H tile issues the TMA copies

  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) mbar_init(&full[i], 1);
    fence_mbar_init();
  }
  for (int i = tid; i < 768; i += kThreads) lut[i] = __ldg(p.lut + i);
  // bytes of the RGB planes past the converted width are only ever multiplied
  // by zero weights (MMA read-ahead); keep them zero, never garbage
  for (int i = tid; i < 6 * CH * SWP / 16; i += kThreads)
    reinterpret_cast<uint4*>(rgb)[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();

  const int total = p.npairs * p.nstrips * p.gh2;
  const int i0 = static_cast<int>((static_cast<long long>(blockIdx.x) * total) / gridDim.x);
  const int i1 = static_cast<int>((static_cast<long long>(blockIdx.x + 1) * total) / gridDim.x);

  // ------------------------------------------------------------ compute warps
  // colour items (frame, row, 16-pixel group): at most 2 per thread; their
  // offsets are launch constants (raw stage: Y / UV byte, RGB plane byte)
  const int NQ16 = p.SWPN >> 4;
  const int citems = 2 * CH * NQ16;
  int cy[2], cuv[2], crgb[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int it = tid + e * kComputeThreads;
    const int q = it % NQ16, rowi = it / NQ16, f = rowi >= CH, rr = rowi - f * CH;
    const int xb = 16 * q, sub = xb >> p.bwshift, xo = xb & p.bwmask;
    cy[e] = f * RAWF + (sub * 16 + rr) * p.BW + xo;
    cuv[e] = f * RAWF + 16 * p.BW * p.NX + (sub * 8 + (rr >> 1)) * p.BW + xo;
    crgb[e] = ((f * 3) * CH + rr) * SWP + xb;
  }
  const uint32_t rgb_s = smem_u32(rgb);
  const uint32_t ring_s = smem_u32(ring);
  const uint32_t lut_s = smem_u32(lut);
  // V-pass role: row group vjg, planes [kPlanesPerWarp*vsub, +kPlanesPerWarp)
  const int vjg = warp & 3, vsub = warp >> 2;
  const int j0 = 8 * vjg + 2 * tq;                 // output rows j0, j0+1 of the band
  const bool jok0 = j0 < 28, jok1 = j0 + 1 < 28;   // group 3 covers rows 24..31
  const bool xok1 = g < 6;                         // second column g+8 inside the 14-wide patch
  // token offset of (row j, patch column 0) within a band's token block (R6):
  // row part hm*2*1176 + ph*14
  const int jo0 = (j0 / 14) * 2 * kCols + (j0 % 14) * 14;

  uint32_t seq = 0;
  int cur = i0;
  Run r;
  while (next_run(p, cur, i1, r)) {
    const int X0 = r.strip * p.sw;
    const int SX0 = __ldg(p.hx + X0) & ~15;
    const int npatch = min(p.sw / 14, (p.W2 - X0) / 14);  // valid patches in this strip
    const bool hact = warp < p.htiles;
    // H-pass B fragments of this warp's output tile (constant over the strip)
    const int htile = r.strip * p.htiles + min(warp, p.htiles - 1);
    uint32_t hb[KSH][3][2];
    {
      const uint32_t* f = p.hfr + static_cast<size_t>(htile) * KSH * 3 * 64 + lane * 2;
#pragma unroll
      for (int k = 0; k < KSH; ++k)
#pragma unroll
        for (int pl = 0; pl < 3; ++pl) {
          hb[k][pl][0] = __ldg(f + (k * 3 + pl) * 64);
          hb[k][pl][1] = __ldg(f + (k * 3 + pl) * 64 + 1);
        }
    }
    // A-fragment byte addresses in an RGB plane: rows g, g+8; columns xs + 4t (+16)
    const uint32_t hA0 = rgb_s + g * SWP + (hact ? __ldg(p.hxs + htile) - SX0 : 0) + 4 * tq;
    const uint32_t hA1 = hA0 + 8 * SWP;
    // ring columns of this thread's outputs (2t, 2t+1 of the tile); masked past the strip / frame
    const int ho = warp * kTileN + 2 * tq;
    const bool hst0 = hact && ho < p.sw && X0 + ho < p.W2;
    const bool hst1 = hact && ho + 1 < p.sw && X0 + ho + 1 < p.W2;
    int next_k = r.kfirst;
    // ring words of source rows kfirst*16 + g and + g + 8 (advanced per chunk)
    int hwA = ((r.kfirst * CH) / 4 + (g >> 2)) % p.TRW;
    int hwB = ((r.kfirst * CH) / 4 + 2 + (g >> 2)) % p.TRW;
    // prefill: the run's first kStages chunks (every stage is free: the previous
    // run consumed all it issued, before the barrier that ended its last band)
    if (issuer)
      for (int j = 0; j < kStages && r.kfirst + j < r.klast; ++j)
        issue_chunk(p, r.pair, SX0, r.kfirst + j, raw + ((seq + j) % kStages) * 2 * RAWF, &full[(seq + j) % kStages]);
    for (int hb_ = r.hb0; hb_ < r.hb1; ++hb_) {
      const int yo0 = hb_ * 28;
      const int kneed = min(p.nchunks, (__ldg(p.vx + yo0 + 27) + __ldg(p.vcnt + yo0 + 27) + CH - 1) / CH);
      for (; next_k < kneed; ++next_k, ++seq) {
        const int k = next_k;
        const int buf = seq % kStages;
        const uint8_t* rawb = raw + buf * 2 * RAWF;
        mbar_wait(&full[buf], (seq / kStages) & 1);
        // ---- a5: NV12 -> RGB planes, 16 pixels per item
        auto convert = [&](int oy, int ouv, int orgb, int e) {
            const uint4 Yv = *reinterpret_cast<const uint4*>(rawb + oy);
            const uint4 UVv = *reinterpret_cast<const uint4*>(rawb + ouv);
            uint4 Rv, Gv, Bv;
            yuv2rgb_4(Yv.x, UVv.x, Rv.x, Gv.x, Bv.x, p.ckR, p.ckG, p.ckGv, p.ckB, p.cbR, p.cbG, p.cbB);
            yuv2rgb_4(Yv.y, UVv.y, Rv.y, Gv.y, Bv.y, p.ckR, p.ckG, p.ckGv, p.ckB, p.cbR, p.cbG, p.cbB);
            yuv2rgb_4(Yv.z, UVv.z, Rv.z, Gv.z, Bv.z, p.ckR, p.ckG, p.ckGv, p.ckB, p.cbR, p.cbG, p.cbB);
            yuv2rgb_4(Yv.w, UVv.w, Rv.w, Gv.w, Bv.w, p.ckR, p.ckG, p.ckGv, p.ckB, p.cbR, p.cbG, p.cbB);
            uint8_t* dst = rgb + orgb;
            *reinterpret_cast<uint4*>(dst) = Rv;
            *reinterpret_cast<uint4*>(dst + CH * SWP) = Gv;
            *reinterpret_cast<uint4*>(dst + 2 * CH * SWP) = Bv;
            if (DBG && p.dbg_src != nullptr) {
              const int it = tid + e * kComputeThreads;
              const int q = it % NQ16, rowi = it / NQ16, f = rowi >= CH, rr = rowi - f * CH;
              const int y = k * CH + rr, x = SX0 + 16 * q;
              if (y < p.H) {
                const uint32_t cw[3][4] = {{Rv.x, Rv.y, Rv.z, Rv.w}, {Gv.x, Gv.y, Gv.z, Gv.w}, {Bv.x, Bv.y, Bv.z, Bv.w}};
                const size_t fi = static_cast<size_t>(p.frame_base + 2 * r.pair + f);
                for (int i = 0; i < 16 && x + i < p.W; ++i)
                  for (int c = 0; c < 3; ++c)
                    p.dbg_src[((fi * p.H + y) * p.W + x + i) * 3 + c] = (cw[c][i >> 2] >> (8 * (i & 3))) & 0xFF;
              }
            }
        };
        {
          if constexpr (KSH <= 2) {  // <= 2 items per thread (host-checked), offsets precomputed
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              if (tid + e * kComputeThreads >= citems) break;
              convert(cy[e], cuv[e], crgb[e], e);
            }
          } else {  // very wide resize windows: any number of items
            for (int it = tid; it < citems; it += kComputeThreads) {
              const int q = it % NQ16, rowi = it / NQ16, f = rowi >= CH, rr = rowi - f * CH;
              const int xb = 16 * q, sub = xb >> p.bwshift, xo = xb & p.bwmask;
              convert(f * RAWF + (sub * 16 + rr) * p.BW + xo, f * RAWF + 16 * p.BW * p.NX + (sub * 8 + (rr >> 1)) * p.BW + xo,
                      ((f * 3) * CH + rr) * SWP + xb, (it - tid) / kComputeThreads);
            }
          }
        }
        bar_sync(1, kComputeThreads);              // RGB planes complete; raw stage free
        // refill the stage just converted with chunk k + kStages; the issuing
        // warp owns no H tile, so this runs beside the H pass, off the critical path
        if (issuer && k + kStages < r.klast) issue_chunk(p, r.pair, SX0, k + kStages, raw + buf * 2 * RAWF, &full[buf]);
        // ---- a6: horizontal pass (MMA) -> ring bytes; planes in groups of 3 for ILP
        if (hact) {
          const uint32_t dA = ring_s + (hwA * RS + ho) * 4 + (g & 3);
          const uint32_t dB = ring_s + (hwB * RS + ho) * 4 + (g & 3);
          constexpr int HG = KSH == 1 ? 3 : 2;  // planes interleaved per group (ILP vs registers)
#pragma unroll
          for (int fg = 0; fg < 6; fg += HG) {
            uint32_t a[HG][KSH][4];
#pragma unroll
            for (int e = 0; e < HG; ++e)
#pragma unroll
              for (int kk = 0; kk < KSH; ++kk) {
                const uint32_t po = (fg + e) * CH * SWP + 32 * kk;
                a[e][kk][0] = lds32(hA0 + po);
                a[e][kk][1] = lds32(hA1 + po);
                a[e][kk][2] = lds32(hA0 + po + 16);
                a[e][kk][3] = lds32(hA1 + po + 16);
              }
            int d2[HG][4], d1[HG][4], d0[HG][4];
#pragma unroll
            for (int e = 0; e < HG; ++e) fir_mma_planes<KSH>(d2[e], d1[e], d0[e], a[e], hb);
#pragma unroll
            for (int e = 0; e < HG; ++e) {
              // clip8 (R4): d0,d1 = row g, columns ho, ho+1; d2,d3 = row g+8
              const uint32_t off = (fg + e) * SW * 4;
              uint32_t q[4];
#pragma unroll
              for (int i = 0; i < 4; ++i)
                q[i] = static_cast<uint32_t>(add_min_relu(combine_planes(d2[e][i], d1[e][i], d0[e][i]), 0,
                                                          (1 << 30) - 1)) >> 22;
              if (hst0) {
                sts8(dA + off, q[0]);
                sts8(dB + off, q[2]);
              }
              if (hst1) {
                sts8(dA + off + 4, q[1]);
                sts8(dB + off + 4, q[3]);
              }
            }
          }
        }
        // advance this thread's two ring rows by one chunk (4 words), wrapping
        hwA += 4;
        hwA -= hwA >= p.TRW ? p.TRW : 0;
        hwB += 4;
        hwB -= hwB >= p.TRW ? p.TRW : 0;
        bar_sync(1, kComputeThreads);  // ring rows complete, RGB planes free
      }
      // ---- a7 + a8 + a9: vertical pass (MMA), normalise, patchify
      {
        const int grp = hb_ * 4 + vjg;
        uint32_t vb[KSV][3][2];
        const uint32_t* f = p.vfr + static_cast<size_t>(grp) * KSV * 3 * 64 + lane * 2;
#pragma unroll
        for (int kk = 0; kk < KSV; ++kk)
#pragma unroll
          for (int pl = 0; pl < 3; ++pl) {
            vb[kk][pl][0] = __ldg(f + (kk * 3 + pl) * 64);
            vb[kk][pl][1] = __ldg(f + (kk * 3 + pl) * 64 + 1);
          }
        const int ys = __ldg(p.vys + grp);
        // A rows: columns (g, g+8) of a patch; k = source rows ys + 32kk + 4t (+16)
        uint32_t rb[KSV][2];
        {
          const uint32_t yw = static_cast<uint32_t>(ys) >> 2;
          int w = static_cast<int>(yw - p.TRW * __umulhi(yw, p.trw_magic)) + tq;  // (ys/4) mod TRW
#pragma unroll
          for (int kk = 0; kk < KSV; ++kk) {
            const int wa = w >= p.TRW ? w - p.TRW : w;
            const int wb4 = wa + 4 >= p.TRW ? wa + 4 - p.TRW : wa + 4;
            rb[kk][0] = ring_s + (wa * RS + kPlanesPerWarp * vsub * SW + g) * 4;
            rb[kk][1] = ring_s + (wb4 * RS + kPlanesPerWarp * vsub * SW + g) * 4;
            w = wa + 8;
          }
        }
        // token block of this (pair, band, strip); patch q of the strip starts at
        // column offset (X0 + 14 q): merge block wb = (X0/28) + q/2, sub-block wm = q&1
        // first token row of this pair (R6: a job's pairs are consecutive gh*gw-row blocks)
        const size_t pair_rows = static_cast<size_t>(p.gh2) * p.gw2 * 4;
        using TokT = std::conditional_t<TOK == FC_TOKENS_BF16, uint16_t,
                                        std::conditional_t<TOK == FC_TOKENS_U8, uint8_t, float>>;
        TokT* tpair;
        if (p.tokj != nullptr) {
          const int job = r.pair / p.ppj;
          tpair = static_cast<TokT*>(p.tokj[job]) + static_cast<size_t>(r.pair - job * p.ppj) * pair_rows * kCols;
        } else {
          tpair = static_cast<TokT*>(p.tokens) + static_cast<size_t>(r.pair) * pair_rows * kCols;
        }
        TokT* tb = tpair + (static_cast<size_t>(hb_) * p.gw2 + X0 / 28) * 4 * kCols + jo0 + g;
#pragma unroll
        for (int e = 0; e < kPlanesPerWarp; ++e) {
          // this warp's planes are frame f = vsub, channels c = e (plane index 3f + c)
          const int f = vsub, c = e;
          const uint32_t lutc = lut_s + c * 1024;
          TokT* tp = tb + (c * 2 + f) * 196;
          constexpr int VG = KSV == 1 ? 2 : 1;  // patches interleaved per group
#pragma unroll
          for (int q0 = 0; q0 < kStrip / 14; q0 += VG) {
            if (q0 >= npatch) break;
            uint32_t a[VG][KSV][4];
#pragma unroll
            for (int e2 = 0; e2 < VG; ++e2)
#pragma unroll
              for (int kk = 0; kk < KSV; ++kk) {
                const uint32_t co = (e * SW + 14 * (q0 + e2)) * 4;
                a[e2][kk][0] = lds32(rb[kk][0] + co);
                a[e2][kk][1] = lds32(rb[kk][0] + co + 32);
                a[e2][kk][2] = lds32(rb[kk][1] + co);
                a[e2][kk][3] = lds32(rb[kk][1] + co + 32);
              }
            int d2[VG][4], d1[VG][4], d0[VG][4];
#pragma unroll
            for (int e2 = 0; e2 < VG; ++e2) fir_mma_planes<KSV>(d2[e2], d1[e2], d0[e2], a[e2], vb);
#pragma unroll
            for (int e2 = 0; e2 < VG; ++e2) {
              const int q = q0 + e2;
              if (q >= npatch) break;
              // d0,d1: column g, rows j0, j0+1; d2,d3: column g+8
              uint32_t sv[4];
              uint32_t o[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                sv[i] = static_cast<uint32_t>(
                    add_min_relu(combine_planes(d2[e2][i], d1[e2][i], d0[e2][i]), 0, (1 << 30) - 1));
                if constexpr (TOK == FC_TOKENS_U8)
                  o[i] = sv[i] >> 22;  // the u8 code (NEXT-1 exchange format)
                else
                  o[i] = lds32(lutc + ((sv[i] >> 20) & 0x3FCu));
              }
              TokT* op = tp + (q >> 1) * 4 * kCols + (q & 1) * kCols;  // wb += q/2, wm = q&1
              st_cs_pred(op, o[0], jok0);
              st_cs_pred(op + 14, o[1], jok1);
              st_cs_pred(op + 8, o[2], jok0 && xok1);
              st_cs_pred(op + 22, o[3], jok1 && xok1);
              if (DBG && p.dbg_rs != nullptr) {
                const size_t fi = static_cast<size_t>(p.frame_base + 2 * r.pair + f);
                for (int ee = 0; ee < 4; ++ee) {
                  const int x = X0 + 14 * q + g + ((ee >= 2) ? 8 : 0), j = j0 + (ee & 1);
                  if ((ee < 2 || xok1) && x < p.W2 && j < 28)
                    p.dbg_rs[((fi * p.H2 + yo0 + j) * p.W2 + x) * 3 + c] = sv[ee] >> 22;
                }
              }
            }
          }
        }
      }
      bar_sync(1, kComputeThreads);  // ring may be overwritten by the next chunks
    }
  }
}

// ------------------------------------------------------------------ host side
using KernelFn = void (*)(Params);

// Instances: k-steps (32 source pixels each) of the H-pass and V-pass MMA
// windows.  8 consecutive outputs need KS*32 >= span + 3 (4-byte alignment).
#define FC_INSTANCES(X) \
  X(1, 1) X(1, 2) X(2, 1) X(2, 2) X(2, 3) X(3, 2) X(3, 3) X(4, 2) X(4, 3) X(4, 4) X(1, 3) X(3, 1) X(1, 4) X(4, 1) X(2, 4) X(3, 4)

struct Instance {
  int ksh, ksv;
  KernelFn fn, fn_dbg, fn_bf16, fn_u8;  // fp32 tokens / + parity-test dumps / bf16 tokens / u8 codes
};
#define FC_INST(A, B)                                                                                           \
  {A, B, fc_fused_kernel<A, B, false, FC_TOKENS_F32>, fc_fused_kernel<A, B, true, FC_TOKENS_F32>, \
   fc_fused_kernel<A, B, false, FC_TOKENS_BF16>, fc_fused_kernel<A, B, false, FC_TOKENS_U8>},
static const Instance kInstances[] = {FC_INSTANCES(FC_INST)};
#undef FC_INST
constexpr int kMaxKS = 4;

static fc_status cuda_fail(cudaError_t e, const char* what) {
  return fail(FC_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename T>
static cudaError_t upload(T** dst, const std::vector<T>& v) {
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(dst), std::max<size_t>(v.size(), 1) * sizeof(T));
  if (e != cudaSuccess) return e;
  return cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
}

// Integer Pillow weight of output o at source index src (0 outside the window).
static int32_t weight_at(const AxisTable& t, int o, int src) {
  if (o < 0 || o >= t.out) return 0;
  const int tap = src - t.xmin[o];
  if (tap < 0 || tap >= t.cnt[o]) return 0;
  return t.iw[static_cast<size_t>(o) * t.ksize + tap];
}
static uint32_t weight_byte(int32_t w, int plane) {
  return plane == 2 ? static_cast<uint32_t>(w >> 16) & 0xFFu : (static_cast<uint32_t>(w) >> (8 * plane)) & 0xFFu;
}

// B fragments of m16n8k32 for a group of 8 outputs (H: 8 columns; V: 8 rows of
// a band) whose windows start at source index xs: b_r (r = 0,1) of lane
// (g = lane/4, t = lane%4) holds k = ks*32 + 16 r + 4 t + [0..3] of output g.
static void frag_group(const AxisTable& t, const int (&outs)[8], int xs, int KS, uint32_t* dst) {
  for (int ks = 0; ks < KS; ++ks)
    for (int pl = 0; pl < 3; ++pl)
      for (int lane = 0; lane < 32; ++lane)
        for (int rr = 0; rr < 2; ++rr) {
          const int g = lane >> 2, tq = lane & 3;
          uint32_t word = 0;
          for (int bb = 0; bb < 4; ++bb) {
            const int k = ks * 32 + 16 * rr + 4 * tq + bb;
            word |= weight_byte(weight_at(t, outs[g], xs + k), pl) << (8 * bb);
          }
          dst[((ks * 3 + pl) * 32 + lane) * 2 + rr] = word;
        }
}

// Span (in k) that a group of outputs needs from its 4-aligned start.
static int group_ks(const AxisTable& t, const int (&outs)[8], int xs) {
  int end = xs;
  for (int g = 0; g < 8; ++g)
    if (outs[g] >= 0 && outs[g] < t.out) end = std::max(end, t.xmin[outs[g]] + t.cnt[outs[g]]);
  return (end - xs + 31) / 32;
}

struct MmaTables {
  int ksh = 1, ksv = 1;
  std::vector<int32_t> hxs, vys;
  std::vector<uint32_t> hfr, vfr;
};

// H: per strip of 84 columns, 11 tiles of 8 consecutive output columns (the
// last tile's columns 84..87 belong to the next strip and carry no weights);
// V: per band, 4 groups of 8 output rows (rows 28hb + 8gi + [0..8), those past
// the band's 28 rows carry no weights).
static void build_mma_tables(const fc_plan_s* P, int sw, MmaTables* m) {
  const AxisTable& th = *P->th;
  const AxisTable& tv = *P->tv;
  const int nstrips = (th.out + sw - 1) / sw;
  const int htiles = (sw + 7) / 8;
  const int nth = nstrips * htiles;
  const int gh2 = tv.out / 28;
  m->hxs.resize(nth);
  m->vys.resize(gh2 * 4);
  auto h_outs = [&](int tt, int (&outs)[8]) {
    const int s = tt / htiles, i = tt % htiles;
    for (int g = 0; g < 8; ++g) {
      const int o = s * sw + 8 * i + g;
      outs[g] = (8 * i + g < sw && o < th.out) ? o : -1;
    }
  };
  auto v_outs = [&](int grp, int (&outs)[8]) {
    const int hb = grp / 4, gi = grp % 4;
    for (int g = 0; g < 8; ++g) outs[g] = (8 * gi + g < 28) ? 28 * hb + 8 * gi + g : -1;
  };
  int ksh = 1, ksv = 1;
  for (int tt = 0; tt < nth; ++tt) {
    int outs[8];
    h_outs(tt, outs);
    const int first = std::min(tt / htiles * sw + 8 * (tt % htiles), th.out - 1);
    m->hxs[tt] = th.xmin[first] & ~3;
    ksh = std::max(ksh, group_ks(th, outs, m->hxs[tt]));
  }
  for (int grp = 0; grp < gh2 * 4; ++grp) {
    int outs[8];
    v_outs(grp, outs);
    m->vys[grp] = tv.xmin[28 * (grp / 4) + 8 * (grp % 4)] & ~3;
    ksv = std::max(ksv, group_ks(tv, outs, m->vys[grp]));
  }
  m->ksh = ksh;
  m->ksv = ksv;
  m->hfr.assign(static_cast<size_t>(nth) * ksh * 3 * 64, 0u);
  m->vfr.assign(static_cast<size_t>(gh2) * 4 * ksv * 3 * 64, 0u);
  for (int tt = 0; tt < nth; ++tt) {
    int outs[8];
    h_outs(tt, outs);
    frag_group(th, outs, m->hxs[tt], ksh, &m->hfr[static_cast<size_t>(tt) * ksh * 3 * 64]);
  }
  for (int grp = 0; grp < gh2 * 4; ++grp) {
    int outs[8];
    v_outs(grp, outs);
    frag_group(tv, outs, m->vys[grp], ksv, &m->vfr[static_cast<size_t>(grp) * ksv * 3 * 64]);
  }
}

// Process-wide cache of uploaded tables, keyed by everything the tables are a
// function of (device, W->W', H->H', normalisation).  Plans of equally shaped
// requests share one upload, so fc_plan + fc_preprocess never touch the device
// synchronously after the first request of a shape.
struct TableKey {
  int dev, sw, w, w2, h, h2;
  uint32_t lut_bits[768];
  bool operator<(const TableKey& o) const { return std::memcmp(this, &o, sizeof(TableKey)) < 0; }
};

static std::mutex g_tables_mu;
static std::map<TableKey, DeviceTables>* g_tables = new std::map<TableKey, DeviceTables>();  // never freed

static fc_status device_tables(fc_plan_s* P, int dev, int sw, DeviceTables** out) {
  std::lock_guard<std::mutex> lk(P->mu);
  const int pkey = dev * 1024 + sw;
  auto it = P->dev.find(pkey);
  if (it != P->dev.end()) {
    *out = &it->second;
    return FC_OK;
  }
  TableKey key;
  std::memset(&key, 0, sizeof(key));
  key.dev = dev;
  key.sw = sw;
  key.w = P->th->in;
  key.w2 = P->th->out;
  key.h = P->tv->in;
  key.h2 = P->tv->out;
  std::memcpy(key.lut_bits, P->lut_dev.data(), sizeof(key.lut_bits));
  std::lock_guard<std::mutex> gk(g_tables_mu);
  auto git = g_tables->find(key);
  if (git != g_tables->end()) {
    *out = &(P->dev[pkey] = git->second);
    return FC_OK;
  }
  MmaTables m;
  build_mma_tables(P, sw, &m);
  if (m.ksh > kMaxKS || m.ksv > kMaxKS)
    return fail(FC_ERR_UNSUPPORTED, "resize window wider than 128 source pixels per 8 outputs");
  DeviceTables t;
  t.ksh = m.ksh;
  t.ksv = m.ksv;
  cudaError_t e = cudaSuccess;
  if (e == cudaSuccess) e = upload(&t.hx, P->th->xmin);
  if (e == cudaSuccess) e = upload(&t.hxs, m.hxs);
  if (e == cudaSuccess) e = upload(&t.hfr, m.hfr);
  if (e == cudaSuccess) e = upload(&t.vx, P->tv->xmin);
  if (e == cudaSuccess) e = upload(&t.vcnt, P->tv->cnt);
  if (e == cudaSuccess) e = upload(&t.vys, m.vys);
  if (e == cudaSuccess) e = upload(&t.vfr, m.vfr);
  if (e == cudaSuccess) e = upload(&t.lut, P->lut_dev);
  if (e != cudaSuccess) {
    cudaFree(t.hx); cudaFree(t.hxs); cudaFree(t.hfr); cudaFree(t.vx); cudaFree(t.vcnt); cudaFree(t.vys);
    cudaFree(t.vfr); cudaFree(t.lut);
    return e == cudaErrorMemoryAllocation ? fail(FC_ERR_OOM, "table upload: out of device memory")
                                          : cuda_fail(e, "table upload");
  }
  (*g_tables)[key] = t;
  *out = &(P->dev[pkey] = t);
  return FC_OK;
}

struct Geometry {
  int sw, htiles, SWPN, SWP, BW, NX, TR, TRW, nstrips, nchunks;
  KernelFn fn, fn_dbg, fn_bf16, fn_u8;
  size_t smem;
};

static size_t smem_bytes(int SWP, int RAWW, int TRW) {
  return 3072 + 128 + static_cast<size_t>(kStages) * 48 * RAWW + static_cast<size_t>(6) * kChunkRows * SWP +
         static_cast<size_t>(TRW) * kRingStride * 4;
}

static fc_status choose_geometry(const fc_plan_s* P, const DeviceTables* dt, int sw, int max_smem, Geometry* g) {
  const int SW = sw;
  g->sw = sw;
  g->htiles = (sw + 7) / 8;
  const auto& th = *P->th;
  const auto& tv = *P->tv;
  const int nstrips = (P->w2 + SW - 1) / SW;
  // per strip: converted width = the taps of its outputs (SWPN); RGB-plane
  // stride = also every MMA tile's 32*KSH-byte read window (SWP)
  int need = 16, taps = 16;
  for (int s = 0; s < nstrips; ++s) {
    const int X0 = s * SW, X1 = std::min(X0 + SW, P->w2);
    const int SX0 = th.xmin[X0] & ~15;
    for (int i = 0; i < g->htiles && X0 + 8 * i < X1; ++i)
      need = std::max(need, (th.xmin[X0 + 8 * i] & ~3) - SX0 + 32 * dt->ksh);
    for (int o = X0; o < X1; ++o) taps = std::max(taps, th.xmin[o] + th.cnt[o] - SX0);
  }
  need = std::max(need, taps);
  // round to an odd multiple of 16 (bank-conflict-free MMA A-fragment loads)
  int swp = (need + 15) / 16;
  if (!(swp & 1)) ++swp;
  g->SWPN = ((taps + 15) / 16) * 16;
  g->SWP = swp * 16;
  g->NX = (g->SWPN + 255) / 256;                       // TMA boxes are at most 256 wide
  g->BW = g->NX == 1 ? g->SWPN : 256;
  // ring depth: after the chunks a band needs (16-row granularity) the ring
  // must still hold the first row of the band's MMA windows
  int tr = 32 * dt->ksv + 16;
  int kmax = 0;
  for (int hb = 0; hb < P->h2 / 28; ++hb) {
    const int ylo = tv.xmin[hb * 28] & ~3;
    const int yend = tv.xmin[hb * 28 + 27] + tv.cnt[hb * 28 + 27];
    const int kneed = (yend + kChunkRows - 1) / kChunkRows;
    tr = std::max(tr, kneed * kChunkRows - ylo);
    kmax = std::max(kmax, kneed);
  }
  g->TR = (tr + 3) & ~3;
  g->TRW = g->TR / 4;
  g->nstrips = nstrips;
  g->nchunks = std::min(kmax, (P->meta.height + kChunkRows - 1) / kChunkRows);
  g->fn = nullptr;
  for (const Instance& in : kInstances)
    if (in.ksh == dt->ksh && in.ksv == dt->ksv) {
      g->fn = in.fn;
      g->fn_dbg = in.fn_dbg;
      g->fn_bf16 = in.fn_bf16;
      g->fn_u8 = in.fn_u8;
    }
  if (!g->fn) return fail(FC_ERR_UNSUPPORTED, "no kernel instance for this resize window");
  if (dt->ksh <= 2 && 2 * kChunkRows * (g->SWPN / 16) > 2 * kComputeThreads)
    return fail(FC_ERR_UNSUPPORTED, "colour stage: more than 2 items per thread");
  g->smem = smem_bytes(g->SWP, g->BW * g->NX, g->TRW);
  if (g->smem > static_cast<size_t>(max_smem))
    return fail(FC_ERR_UNSUPPORTED, "working set exceeds shared memory (resize window too wide)");
  return FC_OK;
}

// ---- TMA tensor maps of the NV12 planes (host-encoded, cached per surface)
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeTiledFn>(nullptr);
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  return fn;
}

struct MapKey {
  uintptr_t ptr;
  int64_t pitch, rows;
  int bw, bh;
  bool operator==(const MapKey& o) const {
    return ptr == o.ptr && pitch == o.pitch && rows == o.rows && bw == o.bw && bh == o.bh;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    return std::hash<uintptr_t>()(k.ptr) ^ (std::hash<int64_t>()(k.pitch * 131 + k.rows) << 1) ^
           (static_cast<size_t>(k.bw) << 20) ^ static_cast<size_t>(k.bh);
  }
};
static std::mutex g_maps_mu;
static std::unordered_map<MapKey, CUtensorMap, MapKeyHash>* g_maps =
    new std::unordered_map<MapKey, CUtensorMap, MapKeyHash>();  // never freed

// 2-D u8 tensor [rows][pitch] with a (bw x bh) box; out-of-bounds -> zeros.
static fc_status tensor_map(const uint8_t* base, int64_t pitch, int64_t rows, int bw, int bh, CUtensorMap* out) {
  const MapKey key{reinterpret_cast<uintptr_t>(base), pitch, rows, bw, bh};
  std::lock_guard<std::mutex> lk(g_maps_mu);
  auto it = g_maps->find(key);
  if (it != g_maps->end()) {
    *out = it->second;
    return FC_OK;
  }
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(FC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(pitch), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(pitch)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(bw), static_cast<cuuint32_t>(bh)};
  const cuuint32_t estr[2] = {1, 1};
  CUtensorMap m;
  const CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_64B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FC_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  if (g_maps->size() > (1u << 16)) g_maps->clear();
  (*g_maps)[key] = m;
  *out = m;
  return FC_OK;
}

// Colour matrix constants (R3, R15): rounded 256x coefficients of the
// standard matrices (include/fc.h), folded into dp2a operand pairs and biases.
static void color_constants(fc_color m, Params* p) {
  struct K { int y, y0, rv, gu, gv, bu; };
  static const K kTab[4] = {
      {298, 16, 409, -100, -208, 516},  // BT.601 limited (R3)
      {298, 16, 459, -55, -136, 541},   // BT.709 limited
      {256, 0, 359, -88, -183, 454},    // BT.601 full
      {256, 0, 403, -48, -120, 475},    // BT.709 full
  };
  const K& k = kTab[static_cast<int>(m)];
  auto pack = [](int hi, int lo) { return (static_cast<uint32_t>(hi & 0xFFFF) << 16) | static_cast<uint32_t>(lo & 0xFFFF); };
  p->ckR = pack(k.rv, k.y);
  p->ckB = pack(k.bu, k.y);
  p->ckG = pack(k.gu, k.y);
  p->ckGv = pack(k.gv, 0);
  p->cbR = -k.y0 * k.y - 128 * k.rv + 128;
  p->cbG = -k.y0 * k.y - 128 * (k.gu + k.gv) + 128;
  p->cbB = -k.y0 * k.y - 128 * k.bu + 128;
}

// The rank's frame list (its sampled frames, then pad copies of the last),
// after validating every surface it reads.  Empty for a rank with no rows.
std::atomic<uint64_t>& launch_counter() {  // fc_kernel_launches(); shared with fc_expand.cu
  static std::atomic<uint64_t> c{0};
  return c;
}

static fc_status rank_frames(const fc_plan_s* P, int32_t rank, const fc_nv12_surface* surfaces, int64_t num_surfaces,
                             std::vector<int64_t>* frames) {
  frames->clear();
  if (rank < 0 || rank >= P->world) return fail(FC_ERR_RANK, "rank outside [0, world_size)");
  const fc_rank_plan& rp = P->ranks[rank].p;
  if (rp.row_end == rp.row_begin) return FC_OK;
  if (!surfaces) return fail(FC_ERR_INVALID_ARG, "surfaces is NULL");
  for (int64_t i = 0; i < rp.sampled_count; ++i) frames->push_back(P->sampled[rp.sampled_begin + i]);
  for (int64_t i = 0; i < rp.pad_frames; ++i) frames->push_back(frames->back());
  const int W = P->meta.width;
  for (int64_t f : *frames) {
    if (f >= num_surfaces) return fail(FC_ERR_MISSING_SURFACE, "surface array too short for frame " + std::to_string(f));
    const fc_nv12_surface& s = surfaces[f];
    if (!s.y || !s.uv) return fail(FC_ERR_MISSING_SURFACE, "NULL surface for frame " + std::to_string(f));
    if ((reinterpret_cast<uintptr_t>(s.y) & 15) || (reinterpret_cast<uintptr_t>(s.uv) & 15))
      return fail(FC_ERR_UNSUPPORTED, "surface planes must be 16-byte aligned");
    if ((s.pitch_y & 15) || (s.pitch_uv & 15) || s.pitch_y < W || s.pitch_uv < W || s.pitch_y > INT32_MAX ||
        s.pitch_uv > INT32_MAX)
      return fail(FC_ERR_UNSUPPORTED, "pitches must be multiples of 16 and >= width");
  }
  return FC_OK;
}

// One launch job: a (plan, rank)'s frame list, its surfaces and its token buffer.
struct Job {
  std::vector<int64_t> frames;
  const fc_nv12_surface* surfaces;
  void* tokens;
};

// ONE persistent launch over every pair of `jobs` (all of P's geometry and
// pair count).  Up to kMaxInlineFrames frames of a single job, the tensor maps
// travel in the kernel parameters (nothing to upload; graph-capturable);
// beyond that, or for several jobs, a descriptor [maps | per-job token bases]
// is copied to a stream-ordered device allocation (cudaMallocAsync, freed
// after the launch in stream order).
static fc_status launch_jobs(fc_plan_s* P, const std::vector<Job>& jobs, void* stream, uint8_t* dbg_src,
                             uint8_t* dbg_rs) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  int major = 0, max_smem = 0, nsm = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (major != 10) return fail(FC_ERR_CUDA, "fc kernels are built for sm_100a only (no CPU/other-arch fallback)");
  const int W = P->meta.width, H = P->meta.height;
  // strips of 2 merge blocks; 1 merge block when a very wide resize window
  // would not fit the working set in shared memory
  DeviceTables* dt = nullptr;
  Geometry g;
  fc_status st = FC_OK;
  for (int sw : {kStrip, 28}) {
    st = device_tables(P, dev, sw, &dt);
    if (st != FC_OK) return st;
    st = choose_geometry(P, dt, sw, max_smem, &g);
    if (st == FC_OK) break;
  }
  if (st != FC_OK) return st;
  const fc_token_dtype td = P->cfg.token_dtype;
  if (td != FC_TOKENS_F32 && (dbg_src || dbg_rs))
    return fail(FC_ERR_UNSUPPORTED, "debug dumps are built for fp32 tokens only");
  KernelFn fn = (dbg_src || dbg_rs)      ? g.fn_dbg
                : td == FC_TOKENS_BF16 ? g.fn_bf16
                : td == FC_TOKENS_U8   ? g.fn_u8
                                       : g.fn;
  e = cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(g.smem));
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kThreads, g.smem);
  if (e != cudaSuccess || occ < 1) return cuda_fail(e, "occupancy query");

  static thread_local Params prm;  // ~31 KB: keep it off the stack
  std::memset(&prm, 0, offsetof(Params, tm));
  prm.W = W;
  prm.H = H;
  prm.W2 = P->w2;
  prm.H2 = P->h2;
  prm.gh2 = static_cast<int>(P->gh / 2);
  prm.gw2 = static_cast<int>(P->gw / 2);
  prm.nstrips = g.nstrips;
  prm.sw = g.sw;
  prm.htiles = g.htiles;
  prm.SWP = g.SWP;
  prm.SWPN = g.SWPN;
  prm.BW = g.BW;
  prm.NX = g.NX;
  prm.bwshift = g.NX == 1 ? 31 : 8;
  prm.bwmask = g.NX == 1 ? -1 : 255;
  prm.TR = g.TR;
  prm.TRW = g.TRW;
  prm.nchunks = g.nchunks;
  prm.hx = dt->hx;
  prm.hxs = dt->hxs;
  prm.hfr = dt->hfr;
  prm.vx = dt->vx;
  prm.vcnt = dt->vcnt;
  prm.vys = dt->vys;
  prm.vfr = dt->vfr;
  prm.lut = dt->lut;
  color_constants(P->cfg.color, &prm);
  prm.dbg_src = dbg_src;
  prm.dbg_rs = dbg_rs;
  prm.trw_magic = static_cast<uint32_t>(((1ull << 32) + g.TRW - 1) / g.TRW);
  const int64_t nfj = static_cast<int64_t>(jobs[0].frames.size());
  const int64_t nf = nfj * static_cast<int64_t>(jobs.size());
  const long long items = (nf / 2) * static_cast<long long>(g.nstrips) * prm.gh2;
  if (items > INT32_MAX) return fail(FC_ERR_UNSUPPORTED, "launch too large (> 2^31 work items)");
  prm.frame_base = 0;
  prm.nframes = static_cast<int>(nf);
  prm.npairs = static_cast<int>(nf / 2);
  prm.ppj = static_cast<int>(nfj / 2);
  prm.tokens = jobs[0].tokens;
  const bool inline_maps = jobs.size() == 1 && nf <= kMaxInlineFrames;
  std::vector<CUtensorMap> maps(inline_maps ? 0 : 2 * nf);
  CUtensorMap* mp = inline_maps ? prm.tm : maps.data();
  for (size_t j = 0; j < jobs.size(); ++j)
    for (int64_t i = 0; i < nfj; ++i) {
      const fc_nv12_surface& sf = jobs[j].surfaces[jobs[j].frames[i]];
      const int64_t fi = static_cast<int64_t>(j) * nfj + i;
      st = tensor_map(sf.y, sf.pitch_y, H, g.BW, kChunkRows, &mp[2 * fi]);
      if (st == FC_OK) st = tensor_map(sf.uv, sf.pitch_uv, H / 2, g.BW, kChunkRows / 2, &mp[2 * fi + 1]);
      if (st != FC_OK) return st;
    }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  void* desc = nullptr;
  if (!inline_maps) {
    const size_t mbytes = maps.size() * sizeof(CUtensorMap);
    const size_t bytes = mbytes + (jobs.size() > 1 ? jobs.size() * sizeof(void*) : 0);
    std::vector<uint8_t> host(bytes);
    std::memcpy(host.data(), maps.data(), mbytes);
    if (jobs.size() > 1)
      for (size_t j = 0; j < jobs.size(); ++j)
        std::memcpy(host.data() + mbytes + j * sizeof(void*), &jobs[j].tokens, sizeof(void*));
    e = cudaMallocAsync(&desc, bytes, s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync (launch descriptor)");
    // pageable source: returns once the bytes are staged, so `host` may die
    e = cudaMemcpyAsync(desc, host.data(), bytes, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) {
      cudaFreeAsync(desc, s);
      return cuda_fail(e, "descriptor upload");
    }
    prm.tmg = reinterpret_cast<const CUtensorMap*>(desc);
    if (jobs.size() > 1) prm.tokj = reinterpret_cast<void* const*>(static_cast<uint8_t*>(desc) + mbytes);
  }
  const int grid = static_cast<int>(std::min<long long>(items, static_cast<long long>(occ) * nsm));
  fn<<<grid, kThreads, g.smem, s>>>(prm);
  e = cudaGetLastError();
  if (desc) cudaFreeAsync(desc, s);
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  return FC_OK;
}

static fc_status preprocess_impl(const fc_plan_t* Pc, int32_t rank, const fc_nv12_surface* surfaces,
                                 int64_t num_surfaces, void* tokens, int64_t grid_thw[3], void* stream,
                                 uint8_t* dbg_src, uint8_t* dbg_rs) {
  if (!Pc) return fail(FC_ERR_INVALID_ARG, "plan is NULL");
  fc_plan_s* P = const_cast<fc_plan_s*>(Pc);
  if (rank < 0 || rank >= P->world) return fail(FC_ERR_RANK, "rank outside [0, world_size)");
  if (grid_thw) {
    grid_thw[0] = P->gt;
    grid_thw[1] = P->gh;
    grid_thw[2] = P->gw;
  }
  std::vector<Job> jobs(1);
  fc_status st = rank_frames(P, rank, surfaces, num_surfaces, &jobs[0].frames);
  if (st != FC_OK || jobs[0].frames.empty()) return st;
  if (!tokens) return fail(FC_ERR_INVALID_ARG, "tokens is NULL");
  jobs[0].surfaces = surfaces;
  jobs[0].tokens = tokens;
  return launch_jobs(P, jobs, stream, dbg_src, dbg_rs);
}

}  // namespace fc

using namespace fc;

extern "C" {

fc_status fc_preprocess(const fc_plan_t* plan, int32_t rank, const fc_nv12_surface* surfaces,
                        int64_t num_surfaces, void* tokens, int64_t grid_thw[3], void* stream) {
  return preprocess_impl(plan, rank, surfaces, num_surfaces, tokens, grid_thw, stream, nullptr, nullptr);
}

fc_status fc_preprocess_debug(const fc_plan_t* plan, int32_t rank, const fc_nv12_surface* surfaces,
                              int64_t num_surfaces, void* tokens, int64_t grid_thw[3], void* stream,
                              uint8_t* rgb_src, uint8_t* rgb_resized) {
  return preprocess_impl(plan, rank, surfaces, num_surfaces, tokens, grid_thw, stream, rgb_src, rgb_resized);
}

fc_status fc_preprocess_batch(const fc_plan_t* const* plans, const int32_t* ranks, int32_t count,
                              const fc_nv12_surface* const* surfaces, const int64_t* num_surfaces,
                              void* const* tokens, void* stream) {
  if (count < 0 || (count > 0 && (!plans || !ranks || !surfaces || !num_surfaces || !tokens)))
    return fail(FC_ERR_INVALID_ARG, "batch arguments");
  // validate every job before any launch; then one launch per maximal run of
  // consecutive jobs sharing source size, resized size and pair count (a
  // homogeneous batch -- config 5 -- is one launch)
  std::vector<Job> jobs(count);
  std::vector<fc_plan_s*> jp(count);
  for (int32_t i = 0; i < count; ++i) {
    if (!plans[i]) return fail(FC_ERR_INVALID_ARG, "batch: plan " + std::to_string(i) + " is NULL");
    jp[i] = const_cast<fc_plan_s*>(plans[i]);
    fc_status st = rank_frames(jp[i], ranks[i], surfaces[i], num_surfaces[i], &jobs[i].frames);
    if (st != FC_OK) return st;
    if (!jobs[i].frames.empty() && !tokens[i]) return fail(FC_ERR_INVALID_ARG, "batch: tokens is NULL");
    jobs[i].surfaces = surfaces[i];
    jobs[i].tokens = tokens[i];
  }
  auto same = [&](int a, int b) {
    const fc_plan_s &A = *jp[a], &B = *jp[b];
    return A.meta.width == B.meta.width && A.meta.height == B.meta.height && A.w2 == B.w2 && A.h2 == B.h2 &&
           A.cfg.token_dtype == B.cfg.token_dtype && A.cfg.color == B.cfg.color && A.lut_dev == B.lut_dev &&
           jobs[a].frames.size() == jobs[b].frames.size();
  };
  std::vector<Job> group;
  for (int32_t i = 0; i < count;) {
    if (jobs[i].frames.empty()) {
      ++i;
      continue;
    }
    int32_t j = i;
    group.clear();
    while (j < count && (jobs[j].frames.empty() || same(i, j))) {
      if (!jobs[j].frames.empty()) group.push_back(jobs[j]);
      ++j;
    }
    fc_status st = launch_jobs(jp[i], group, stream, nullptr, nullptr);
    if (st != FC_OK) return st;
    i = j;
  }
  return FC_OK;
}

uint64_t fc_kernel_launches(void) { return launch_counter().load(std::memory_order_relaxed); }

void fc_plan_destroy(fc_plan_t* P) {
  // device tables belong to the process-wide cache (shared by equal shapes)
  delete P;
}

}  // extern "C"
