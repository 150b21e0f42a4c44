// fc_fused.cuh -- the fused sm_100a kernel of the preprocessing hot path
// (template; instantiated in fc_inst_ks*.cu, launched by fc_kernels.cu).
//
// One launch per rank (or per batch of requests) computes, for each temporal
// pair of the sampled frames (Alg. 1 l.21-22, P:386-389,
// "convert_AVframes_to_tensor_and_resize"):
//   a5  NV12 -> RGB, integer YUV matrix (BT.601 limited by default)  (R3, R15)
//   a6  horizontal Pillow-bicubic pass, u8 intermediate             (R4)
//   a7  vertical Pillow-bicubic pass                                 (R4)
//   a8  rescale + normalise through a 3x256 table                    (R5, R16)
//   a9  temporal pad + 14x14x2 patchify in 2x2 merge order           (R6)
// in ONE pass over HBM: NV12 bytes are read once (plus strip halos), tokens
// are written once.  Work unit: one temporal pair x one strip of 2 merge
// blocks (56 output columns), walking down the frame one merge-block row (28
// output rows, a "band") at a time.  Source rows are converted and
// horizontally filtered once each into a ring of u8 rows (column-major, so
// that 4 vertically adjacent taps are one 32-bit word); the vertical pass
// reads the ring.  Both resize passes are exact int8 tensor-core MMAs
// (mma.sync m16n8k32, u8 x s8/u8 -> s32) on byte planes of Pillow's 22-bit
// weights: sum px*iw = ((D2 << 8) + D1) << 8 + D0.  DESIGN.md section 6.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "fc_device.cuh"
#include "fc_internal.h"

namespace fc {

#ifndef FC_HG2
#define FC_HG2 2  // the same for wide windows (KSH > 1)
#endif
#ifndef FC_LB_NARROW
#define FC_LB_NARROW 4  // min CTAs/SM of the narrow-window instances (64 registers; A/B knob)
#endif
#ifndef FC_LB_WIDE
#define FC_LB_WIDE 3  // min CTAs/SM the wide-window instances are compiled for (register cap; A/B knob)
#endif
// FC_CHECKED=1 builds (tools/checked_build.sh): every shared-memory and token
// address the kernel forms is range-checked and a violation traps -- the
// bounds evidence compute-sanitizer no longer provides on the GPU pool.
#ifndef FC_CHECKED
#define FC_CHECKED 0
#endif
#if FC_CHECKED
#include <cstdio>
#define FC_CHK(c, what)                                                                          \
  do {                                                                                           \
    if (!(c)) {                                                                                  \
      printf("fc check failed: %s (block %d thread %d)\n", what, blockIdx.x, threadIdx.x);      \
      __trap();                                                                                  \
    }                                                                                            \
  } while (0)
#else
#define FC_CHK(c, what) \
  do {                  \
  } while (0)
#endif
#ifndef FC_VG1
#define FC_VG1 1  // V pass: patches per MMA group for KSV = 1 (A/B knob)
#endif
#ifndef FC_BAND_BAR
#define FC_BAND_BAR 0  // CTA barrier after every band's V pass (redundant; A/B knob)
#endif
#ifndef FC_COLOR_C
#define FC_COLOR_C 1  // narrow windows: colour with chroma terms per chroma pair (yuv2rgb_4x2c; A/B knob)
#endif
#ifndef FC_PREF_VB
#define FC_PREF_VB 0  // L1 prefetch of the band's V fragments at the band start (A/B knob)
#endif
#ifndef FC_PREF
#define FC_PREF 1  // per-band table reads issued a band ahead (A/B knob)
#endif
#ifndef FC_HG1
#define FC_HG1 2  // H-pass planes interleaved per MMA group, narrow windows (A/B: 2 beats 3 by 1% on c2, 6 spills)
#endif
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
// normalisation table in shared memory: per channel, entries for v in
// [-kLutLo, 256 + kLutLo), the entries outside [0, 255] repeating LUT[0] /
// LUT[255] -- so the V pass indexes it with floor(S / 2^22) and clip8's clamp
// disappears (the host checks every V output row's reachable range fits)
constexpr int kLutLo = 48;
constexpr int kLutN = 256 + 2 * kLutLo;                      // 352 entries per channel
constexpr int kLutBytes = (3 * kLutN * 4 + 127) / 128 * 128;  // 4224: keeps the TMA stages 128-B aligned
constexpr int kMaxStages = 4;              // raw NV12 chunk buffers: p.nstages in {2, 4} (host-chosen)
constexpr int kIssueWarp = kComputeWarps - 1;  // owns no H-pass tile (7 tiles of 8 cover a 56-column strip)
static_assert((kStrip + kTileN - 1) / kTileN < kComputeWarps, "the TMA issuing warp must own no H tile");

struct Params {
  int W, H, W2, H2;
  int gh2, gw2;       // merge blocks per column / row
  int nstrips, npairs;
  int sw, htiles;      // strip width (84 or 28 output columns), H tiles per strip
  int SWP;            // RGB-plane row stride (8 mod 16)
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
  int nstages, stage_shift;  // raw TMA stages (2 or 4; the host trades pipeline depth for CTAs/SM) and log2
  // NEXT-2 paged output (PAGED instances): token row i of this launch goes to
  // pool row page_ids[(page_first + i) >> page_shift] * page_rows + ((page_first + i) & page_mask)
  const int32_t* page_ids;  // device (launch descriptor)
  long long page_first;     // pv_cu_page_len mod page_rows (slot of the launch's first row)
  uint32_t page_shift, page_mask, page_rows;
  void* const* tokj;  // device: per-job token base (batch launches) or null -> tokens
  const CUtensorMap* tmg;  // device copy of the maps (launches past kMaxInlineFrames frames) or null -> tm
  unsigned long long* cta_t;  // FC_CTA_TIMES experiments: per CTA {start, end, smid} (ns) or null
  int smap;           // 1: strip-synchronous work mapping (CTA b owns strip b % nstrips)
  int sxmask;         // strip source-window start alignment: ~15, or ~31 for I420 (TMA box starts 16-B aligned)
  // NEXT-1 column-split output (COLS instances): token (row i, column col) goes to
  // tokens[b * cs_bstride + i * cs_C + col - b * cs_C], b = col / cs_C = umulhi(col, cs_magic)
  long long cs_bstride;  // elements per column block (rows of the launch x cs_C)
  int cs_C;              // columns per block: 1176 / world_size
  uint32_t cs_magic;     // ceil(2^32 / cs_C)
  // tensor maps per frame: Y (box BW x 16) + UV (box BW x 8) for NV12, or
  // Y + U + V (boxes BW/2 x 8) for I420 -- up to 2 * kMaxInlineFrames maps inline
  CUtensorMap tm[2 * kMaxInlineFrames];
};

// Walk of one CTA's work: contiguous (pair, strip, band) items, split into
// runs that stay inside one (pair, strip).
struct Run {
  int pair, strip, hb0, hb1, kfirst, klast;
};

__device__ __forceinline__ bool next_run(const Params& p, int& cur, int i1, int sfix, Run& r) {
  if (cur >= i1) return false;
  const int ps = cur / p.gh2;
  r.hb0 = cur - ps * p.gh2;
  if (sfix >= 0) {  // strip-synchronous mapping: cur walks (pair, band) of strip sfix
    r.pair = ps;
    r.strip = sfix;
  } else {
    r.pair = ps / p.nstrips;
    r.strip = ps - r.pair * p.nstrips;
  }
  r.hb1 = min(p.gh2, r.hb0 + (i1 - cur));
  cur += r.hb1 - r.hb0;
  r.kfirst = (__ldg(p.vx + 28 * r.hb0) & ~3) / kChunkRows;
  r.klast = min(p.nchunks, (__ldg(p.vx + 28 * r.hb1 - 1) + __ldg(p.vcnt + 28 * r.hb1 - 1) + kChunkRows - 1) / kChunkRows);
  return true;
}

// Raw-stage byte offset of the chroma of (sub-box, luma row rr, byte column xo
// within the sub-box): NV12 -> the interleaved U,V pair row; I420 -> the U row
// (the V row is 4*BW bytes further)
template <bool I420>
__device__ __forceinline__ int chroma_offset(const Params& p, int base, int sub, int rr, int xo) {
  return I420 ? base + sub * 8 * p.BW + (rr >> 1) * (p.BW >> 1) + (xo >> 1)
                : base + (sub * 8 + (rr >> 1)) * p.BW + xo;
}

// Issue the TMA tensor copies of one 16-row chunk into a raw stage (one
// thread): per frame of the pair, NX boxes of Y (BW x 16 rows) then NX boxes
// of UV (BW x 8 rows), after arming the stage's full barrier with their bytes.
template <bool I420>
__device__ __forceinline__ void issue_chunk(const Params& p, int pair, int SX0, int k, uint8_t* raw, uint64_t* bar) {
  const CUtensorMap* tm = p.tmg != nullptr ? p.tmg : p.tm;
  constexpr int mpf = I420 ? 3 : 2;  // maps per frame: Y, UV (NV12) or Y, U, V (I420)
  fence_proxy_async();
  mbar_arrive_expect_tx(bar, static_cast<uint32_t>(2 * 24 * p.BW * p.NX));
  for (int f = 0; f < 2; ++f)
    for (int pl = 0; pl < 2; ++pl)
      for (int sub = 0; sub < p.NX; ++sub) {
        uint8_t* dst = raw + f * 24 * p.BW * p.NX + (pl ? 16 * p.BW * p.NX + sub * 8 * p.BW : sub * 16 * p.BW);
        const CUtensorMap* m = &tm[mpf * (2 * pair + f) + pl];
        if (pl && I420) {  // U rows then V rows, BW/2 bytes each, in the sub-box's 8*BW bytes
          tma_load_2d(dst, m, (SX0 >> 1) + sub * (p.BW >> 1), k * (kChunkRows / 2), bar);
          tma_load_2d(dst + 4 * p.BW, m + 1, (SX0 >> 1) + sub * (p.BW >> 1), k * (kChunkRows / 2), bar);
        } else {
          tma_load_2d(dst, m, SX0 + sub * p.BW, pl ? k * (kChunkRows / 2) : k * kChunkRows, bar);
        }
      }
}

// Persistent fused kernel, 8 warps, 4 CTAs/SM (narrow windows) or 2-3.  Per
// 16-row chunk:
//   lane 0 of warp 7 refills the raw stage just converted with the chunk
//       nstages ahead (2-D TMA, mbarrier expect_tx) beside the H pass;
//   all warps: a5 colour (dp2a), items of 8 px x 2 rows -> row-pair
//       interleaved RGB planes; barrier;
//   warps 0..6: a6 horizontal pass, warp w owns output tile w (8 columns) of
//       the strip; three byte-plane MMAs per 16 rows x 8 outputs (MMA rows
//       g / g+8 = the two rows of row pair (g>>1)|(g&1)<<2, A fragment = one
//       LDS.128) -> saturating pack -> u8 ring (4 source rows per 32-bit word,
//       one 16-bit store per column pair); barrier.
// Per band: a7 vertical pass, warp w owns 8-row group (w&3) and the three
// channels of frame w>>2; one MMA tile per 14-column patch, then a8 table +
// a9 patch-order stores; barrier.
// Work items are (pair, strip, band) triples; CTA b takes [b*T/G, (b+1)*T/G).
// Strips are whole merge blocks, so every token row is written by one CTA in
// one band (no partial-sector merging across CTAs in L2).
template <int KSH, int KSV, bool DBG, int TOK, bool PAGED = false, bool I420 = false, bool COLS = false>
// Narrow-window instances (KSH = KSV = 1: c2, c3, c5) fit 64 registers without
// spills and run 4 CTAs/SM (with 2 TMA stages); wider windows keep 80 / 3.
__global__ void __launch_bounds__(kThreads, (KSH == 1 && KSV == 1) ? FC_LB_NARROW : FC_LB_WIDE)
    fc_fused_kernel(const __grid_constant__ Params p) {
  constexpr int SW = kStrip;
  constexpr int CH = kChunkRows;
  constexpr int RS = kRingStride;

  extern __shared__ __align__(1024) uint8_t smem[];
  uint32_t* lut = reinterpret_cast<uint32_t*>(smem);              // 3 x 256 token bits at offset 0
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kLutBytes);  // nstages full barriers
  const int RAWF = 24 * p.BW * p.NX;                              // raw bytes per frame per stage
  uint8_t* raw = smem + kLutBytes + 128;                          // [nstages][2 f][Y boxes | UV boxes]
  const int NS = p.nstages;
  const uint32_t smask = static_cast<uint32_t>(NS - 1);
  const int SWP = p.SWP;
  // RGB planes [2 f][3 c][8 row pairs][2 SWP]: a row pair interleaves its two
  // rows in 4-byte column groups, (row r, column x) at (r/2)*2SWP + (x/4)*8 +
  // (r&1)*4 + x%4, so one LDS.128 is a whole H-pass A fragment
  uint8_t* rgb = raw + NS * 2 * RAWF;
  uint32_t* ring = reinterpret_cast<uint32_t*>(rgb + 6 * CH * SWP);  // [TRW][RS] words: [w][f][c][x]

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tq = lane & 3;
  const bool issuer = tid == kIssueWarp * 32;  // lane 0 of the warp without an H tile issues the TMA copies

  if (tid == 0) {
    if (p.cta_t != nullptr) p.cta_t[3 * blockIdx.x] = globaltimer();
    for (int i = 0; i < NS; ++i) mbar_init(&full[i], 1);
    fence_mbar_init();
  }
  for (int i = tid; i < 3 * kLutN; i += kThreads) lut[i] = __ldg(p.lut + i);
  // bytes of the RGB planes past the converted width are only ever multiplied
  // by zero weights (MMA read-ahead); keep them zero, never garbage
  for (int i = tid; i < 6 * CH * SWP / 16; i += kThreads)
    reinterpret_cast<uint4*>(rgb)[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  // (PDL) the prologue above only reads the plan's constant tables; the NV12
  // surfaces, launch descriptor and token buffer may belong to the previous
  // launch on the stream, so everything below waits for it; the next launch
  // may begin its own prologue as soon as this one's CTAs start retiring
  grid_launch_dependents();
  grid_dependency_wait();

  const int total = p.npairs * p.nstrips * p.gh2;
  int i0 = static_cast<int>((static_cast<long long>(blockIdx.x) * total) / gridDim.x);
  int i1 = static_cast<int>((static_cast<long long>(blockIdx.x + 1) * total) / gridDim.x);
  // strip-synchronous mapping: CTA b owns strip b % nstrips over the (pair,
  // band) range of group b / nstrips, so the nstrips CTAs of a group walk
  // side by side down the same frames and share their strip halos in L2
  int sfix = -1;
  // (grid = G: the first r strips get Qhi = ceil(G / nstrips) groups, the
  // others Qhi - 1, so only the r / nstrips boundary drifts)
  if (p.smap) {
    const int ns = p.nstrips, q = blockIdx.x / ns;
    sfix = blockIdx.x - q * ns;
    const int qhi = (gridDim.x + ns - 1) / ns, rr = gridDim.x - (qhi - 1) * ns;
    const int Q = sfix < rr ? qhi : qhi - 1;
    const long long PB = static_cast<long long>(p.npairs) * p.gh2;
    i0 = static_cast<int>(q * PB / Q);
    i1 = static_cast<int>((q + 1) * PB / Q);
  }

  // ------------------------------------------------------------ compute warps
  // colour items (frame, row pair, 8-pixel group): 16 pixels sharing 4 chroma
  // pairs, at most 2 items per thread; their offsets are launch constants
  // (raw stage: even-row Y / UV byte, RGB plane byte)
  const int NQ8 = p.SWPN >> 3;
  const int citems = 2 * (CH / 2) * NQ8;
  int cy[2], cuv[2], crgb[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int it = tid + e * kComputeThreads;
    const int q = it % NQ8, rowi = it / NQ8, f = rowi >= CH / 2, rp = rowi - f * (CH / 2);
    const int xb = 8 * q, sub = xb >> p.bwshift, xo = xb & p.bwmask;
    cy[e] = f * RAWF + (sub * 16 + 2 * rp) * p.BW + xo;
    cuv[e] = chroma_offset<I420>(p, f * RAWF + 16 * p.BW * p.NX, sub, 2 * rp, xo);
    crgb[e] = (f * 3) * CH * SWP + rp * 2 * SWP + 2 * xb;
  }
  const uint32_t rgb_s = smem_u32(rgb);
  const uint32_t ring_s = smem_u32(ring);
  const uint32_t lut_s = smem_u32(lut);
  // V-pass role: row group vjg, planes [kPlanesPerWarp*vsub, +kPlanesPerWarp)
  const int vjg = warp & 3, vsub = warp >> 2;
  // MMA N columns 2t / 2t+1 are output rows t / t+4 of the 8-row group (the host
  // orders the V weights so), so each LUT load of a warp reads a compact 4-row
  // footprint: fewer distinct values per bank, fewer shared-memory conflicts
  const int j0 = 8 * vjg + tq, j1 = j0 + 4;        // this thread's output rows of the band
  const bool jok0 = j0 < 28, jok1 = j1 < 28;       // group 3 covers rows 24..31
  // V-pass MMA rows g / g+8 are patch columns 2g / 2g+1: one LDS.64 loads both
  // A words (adjacent ring columns) and one 8-byte store writes both outputs
  const bool xok = g < 7;                          // columns 2g, 2g+1 inside the 14-wide patch
  // token offset of (row j, patch column 0) within a band's token block (R6):
  // row part hm*2*1176 + ph*14
  const int jo0 = (j0 / 14) * 2 * kCols + (j0 % 14) * 14;
  const int djo = (j1 / 14) * 2 * kCols + (j1 % 14) * 14 - jo0;  // row j1 relative to row j0 (other half at 14)

  uint32_t seq = 0;
  Run r;
  int cur = i0;
  while (next_run(p, cur, i1, sfix, r)) {
    const int X0 = r.strip * p.sw;
    const int SX0 = __ldg(p.hx + X0) & p.sxmask;  // 16-aligned (NV12) / 32-aligned (I420: U, V boxes at SX0/2)
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
    // A-fragment address in an RGB plane.  H-pass MMA rows g / g+8 are the two
    // source rows of row pair hp = (g>>1) | (g&1)<<2: a thread's two rows of one
    // output column are the two bytes of one ring half-word, and the two row
    // pairs of a quarter-warp's LDS.128 lie 64 B apart mod 128 (row-pair stride
    // 2SWP = 16 mod 32): no bank conflicts.  The MMA's K order is permuted (the
    // host orders the B fragments so): thread t's k = 4t..4t+3 and 16+4t.. are
    // source columns xs + 8t + [0, 8), i.e. a0 a1 a2 a3 = 16 contiguous bytes.
    const int hp = (g >> 1) | ((g & 1) << 2);
    const uint32_t hA = rgb_s + hp * 2 * SWP + 2 * (hact ? __ldg(p.hxs + htile) - SX0 : 0) + 16 * tq;
    // ring columns of this thread's outputs (2t, 2t+1 of the tile); masked past the strip / frame
    const int ho = warp * kTileN + 2 * tq;
    const bool hst0 = hact && ho < p.sw && X0 + ho < p.W2;
    const bool hst1 = hact && ho + 1 < p.sw && X0 + ho + 1 < p.W2;
    int next_k = r.kfirst;
    // ring word of source rows kfirst*16 + 2hp, 2hp + 1 (advanced per chunk)
    int hwA = ((r.kfirst * CH) / 4 + (hp >> 1)) % p.TRW;
    // prefill: the run's first nstages chunks (every stage is free: the previous
    // run consumed all it issued, before the barrier that ended its last band)
    if (issuer)
      for (int j = 0; j < NS && r.kfirst + j < r.klast; ++j)
        issue_chunk<I420>(p, r.pair, SX0, r.kfirst + j, raw + ((seq + j) & smask) * 2 * RAWF, &full[(seq + j) & smask]);
#if FC_PREF
    // per-band table reads are issued one band ahead (their L2 latency was
    // exposed at every band start): the end row of the band's last V window
    int vend_nx = __ldg(p.vx + 28 * r.hb0 + 27) + __ldg(p.vcnt + 28 * r.hb0 + 27);
#endif
    for (int hb_ = r.hb0; hb_ < r.hb1; ++hb_) {
      const int yo0 = hb_ * 28;
#if FC_PREF
      const int kneed = min(p.nchunks, (vend_nx + CH - 1) / CH);
      if (hb_ + 1 < r.hb1) vend_nx = __ldg(p.vx + yo0 + 55) + __ldg(p.vcnt + yo0 + 55);
      const int ys_pf = __ldg(p.vys + hb_ * 4 + vjg);  // consumed by this band's V pass, after the chunks
#if FC_PREF_VB
      // the warp's V weight fragments of this band (KSV*3 blocks of 256 B): one
      // L1 prefetch per 128-B line, so the V pass's fragment loads hit L1
      if (lane < KSV * 6)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(p.vfr + static_cast<size_t>(hb_ * 4 + vjg) * KSV * 3 * 64 + lane * 32));
#endif
#else
      const int kneed = min(p.nchunks, (__ldg(p.vx + yo0 + 27) + __ldg(p.vcnt + yo0 + 27) + CH - 1) / CH);
#endif
      for (; next_k < kneed; ++next_k, ++seq) {
        const int k = next_k;
        const int buf = seq & smask;
        const uint8_t* rawb = raw + buf * 2 * RAWF;
        mbar_wait(&full[buf], (seq >> p.stage_shift) & 1);
        // ---- a5: NV12 -> RGB planes, 8 pixels x 2 rows per item
        auto convert = [&](int oy, int ouv, int orgb, int e) {
            FC_CHK(oy >= 0 && oy + p.BW + 8 <= 2 * RAWF && ouv >= 0 && ouv + (I420 ? 4 * p.BW + 4 : 8) <= 2 * RAWF,
                   "colour raw read outside its stage");
            FC_CHK(orgb >= 0 && orgb + 2 * CH * SWP + 16 <= 6 * CH * SWP, "colour store outside the RGB planes");
            const uint2 Ye = *reinterpret_cast<const uint2*>(rawb + oy);          // even row, 8 pixels
            const uint2 Yo = *reinterpret_cast<const uint2*>(rawb + oy + p.BW);   // odd row
            uint2 UVv;
            if constexpr (I420) {  // interleave 4 U and 4 V bytes into NV12 order [U0 V0 U1 V1 ...]
              const uint32_t u = *reinterpret_cast<const uint32_t*>(rawb + ouv);
              const uint32_t v = *reinterpret_cast<const uint32_t*>(rawb + ouv + 4 * p.BW);
              UVv = make_uint2(__byte_perm(u, v, 0x5140), __byte_perm(u, v, 0x7362));
            } else {
              UVv = *reinterpret_cast<const uint2*>(rawb + ouv);
            }
            // per channel: even row px 0-3, odd row px 0-3, even px 4-7, odd px 4-7
            uint4 Rv, Gv, Bv;
            if constexpr (FC_COLOR_C && KSH == 1) {  // c2 -0.5%; c4 (KSH = 2) +1.2%, so wide windows keep 4x2
            yuv2rgb_4x2c(Ye.x, Yo.x, UVv.x, Rv.x, Gv.x, Bv.x, Rv.y, Gv.y, Bv.y, p.ckR, p.ckG, p.ckGv, p.ckB, p.cbR,
                         p.cbG, p.cbB);
            yuv2rgb_4x2c(Ye.y, Yo.y, UVv.y, Rv.z, Gv.z, Bv.z, Rv.w, Gv.w, Bv.w, p.ckR, p.ckG, p.ckGv, p.ckB, p.cbR,
                         p.cbG, p.cbB);
            } else {
            yuv2rgb_4x2(Ye.x, Yo.x, UVv.x, Rv.x, Gv.x, Bv.x, Rv.y, Gv.y, Bv.y, p.ckR, p.ckG, p.ckGv, p.ckB, p.cbR,
                        p.cbG, p.cbB);
            yuv2rgb_4x2(Ye.y, Yo.y, UVv.y, Rv.z, Gv.z, Bv.z, Rv.w, Gv.w, Bv.w, p.ckR, p.ckG, p.ckGv, p.ckB, p.cbR,
                        p.cbG, p.cbB);
            }
            uint8_t* dst = rgb + orgb;  // 16-byte aligned (row-pair stride 2SWP = 0 mod 16)
            *reinterpret_cast<uint4*>(dst) = Rv;
            *reinterpret_cast<uint4*>(dst + CH * SWP) = Gv;
            *reinterpret_cast<uint4*>(dst + 2 * CH * SWP) = Bv;
            if (DBG && p.dbg_src != nullptr) {
              const int it = tid + e * kComputeThreads;
              const int q = it % NQ8, rowi = it / NQ8, f = rowi >= CH / 2, rp = rowi - f * (CH / 2);
              const uint32_t cw[3][4] = {{Rv.x, Rv.y, Rv.z, Rv.w}, {Gv.x, Gv.y, Gv.z, Gv.w}, {Bv.x, Bv.y, Bv.z, Bv.w}};
              const size_t fi = static_cast<size_t>(p.frame_base + 2 * r.pair + f);
              for (int h = 0; h < 2; ++h) {
                const int y = k * CH + 2 * rp + h, x = SX0 + 8 * q;
                if (y < p.H)
                  for (int i = 0; i < 8 && x + i < p.W; ++i)
                    for (int c = 0; c < 3; ++c)
                      p.dbg_src[((fi * p.H + y) * p.W + x + i) * 3 + c] =
                          (cw[c][2 * (i >> 2) + h] >> (8 * (i & 3))) & 0xFF;
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
              const int q = it % NQ8, rowi = it / NQ8, f = rowi >= CH / 2, rp = rowi - f * (CH / 2);
              const int xb = 8 * q, sub = xb >> p.bwshift, xo = xb & p.bwmask;
              convert(f * RAWF + (sub * 16 + 2 * rp) * p.BW + xo,
                      chroma_offset<I420>(p, f * RAWF + 16 * p.BW * p.NX, sub, 2 * rp, xo),
                      (f * 3) * CH * SWP + rp * 2 * SWP + 2 * xb, (it - tid) / kComputeThreads);
            }
          }
        }
        bar_sync(1, kComputeThreads);              // RGB planes complete; raw stage free
        // refill the stage just converted with chunk k + nstages; the issuing
        // warp owns no H tile, so this runs beside the H pass, off the critical path
        if (issuer && k + NS < r.klast) issue_chunk<I420>(p, r.pair, SX0, k + NS, raw + buf * 2 * RAWF, &full[buf]);
        // ---- a6: horizontal pass (MMA) -> ring bytes; planes in groups of HG for ILP
        if (hact) {
          const uint32_t dA = ring_s + (hwA * RS + ho) * 4 + 2 * (hp & 1);  // bytes of rows 2hp, 2hp+1
          constexpr int HG = KSH == 1 ? FC_HG1 : FC_HG2;  // planes interleaved per group (ILP vs registers)
#pragma unroll
          for (int fg = 0; fg < 6; fg += HG) {
            uint32_t a[HG][KSH][4];
#pragma unroll
            for (int e = 0; e < HG; ++e)
#pragma unroll
              for (int kk = 0; kk < KSH; ++kk) {
                FC_CHK(hA + (fg + e) * CH * SWP + 64 * kk >= rgb_s &&
                           hA + (fg + e) * CH * SWP + 64 * kk + 16 <= rgb_s + 6 * CH * SWP,
                       "H A fragment outside the RGB planes");
                lds128(a[e][kk], hA + (fg + e) * CH * SWP + 64 * kk);  // k-step kk: 32 columns x 2 rows
              }
            int d2[HG][4], d1[HG][4], d0[HG][4];
#pragma unroll
            for (int e = 0; e < HG; ++e) fir_mma_planes<KSH>(d2[e], d1[e], d0[e], a[e], hb);
#pragma unroll
            for (int e = 0; e < HG; ++e) {
              // clip8 (R4) = sat_u8(S >> 22) (arithmetic shift; S < 2^31 by Pillow's
              // headroom): d0,d1 = row 2hp, columns ho, ho+1; d2,d3 = row 2hp+1
              const uint32_t off = (fg + e) * SW * 4;
              int v[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) v[i] = combine_planes(d2[e][i], d1[e][i], d0[e][i]) >> 22;
              FC_CHK(!hst0 || (dA + off >= ring_s && dA + off + 2 <= ring_s + p.TRW * RS * 4), "H ring store outside the ring");
              FC_CHK(!hst1 || (dA + off + 4 >= ring_s && dA + off + 6 <= ring_s + p.TRW * RS * 4), "H ring store outside the ring");
              if (hst0) sts16(dA + off, pack_sat_u8(v[2], v[0], 0u));      // column ho: rows 2hp, 2hp+1
              if (hst1) sts16(dA + off + 4, pack_sat_u8(v[3], v[1], 0u));  // column ho + 1
            }
          }
        }
        // advance this thread's ring row word by one chunk (4 words), wrapping
        hwA += 4;
        hwA -= hwA >= p.TRW ? p.TRW : 0;
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
#if FC_PREF
        const int ys = ys_pf;
#else
        const int ys = __ldg(p.vys + grp);
#endif
        // A rows: columns (g, g+8) of a patch; k = source rows ys + 32kk + 4t (+16)
        uint32_t rb[KSV][2];
        {
          const uint32_t yw = static_cast<uint32_t>(ys) >> 2;
          int w = static_cast<int>(yw - p.TRW * __umulhi(yw, p.trw_magic)) + tq;  // (ys/4) mod TRW
#pragma unroll
          for (int kk = 0; kk < KSV; ++kk) {
            const int wa = w >= p.TRW ? w - p.TRW : w;
            const int wb4 = wa + 4 >= p.TRW ? wa + 4 - p.TRW : wa + 4;
            rb[kk][0] = ring_s + (wa * RS + kPlanesPerWarp * vsub * SW + 2 * g) * 4;
            rb[kk][1] = ring_s + (wb4 * RS + kPlanesPerWarp * vsub * SW + 2 * g) * 4;
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
        TokT* tb = tpair + (static_cast<size_t>(hb_) * p.gw2 + X0 / 28) * 4 * kCols + jo0 + 2 * g;
        // paged output: the pool row of each patch's token row (merge block q/2,
        // sub-block q&1, this thread's half hm = j0/14) -- SPEC write_chunk mapping
        uint32_t prow[2][4];  // [row j0 / j1][patch]
        if constexpr (PAGED) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const long long row0 = static_cast<long long>(r.pair) * static_cast<long long>(pair_rows) +
                                   (static_cast<long long>(hb_) * p.gw2 + X0 / 28) * 4 + ((h ? j1 : j0) / 14) * 2;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const long long sl = p.page_first + row0 + (q >> 1) * 4 + (q & 1);
              // only rows this thread stores: rows 28..31 of group 3 (jok false) may lie past
              // the write's last page (page_ids[num_pages] read)
              const bool live = q < npatch && (h ? jok1 : jok0);
              prow[h][q] = live ? static_cast<uint32_t>(__ldg(p.page_ids + (sl >> p.page_shift))) * p.page_rows +
                                      static_cast<uint32_t>(sl & p.page_mask)
                                : 0u;
            }
          }
        }
#pragma unroll
        for (int e = 0; e < kPlanesPerWarp; ++e) {
          // this warp's planes are frame f = vsub, channels c = e (plane index 3f + c)
          const int f = vsub, c = e;
          const uint32_t lutc = lut_s + (c * kLutN + kLutLo) * 4;  // entry of v = 0
          TokT* tp = tb + (c * 2 + f) * 196;
          // patches per MMA group: 2 for KSV = 2 (c4 -2.9%), 1 for narrow windows (2: c2 +0.4%; 4 spills)
          constexpr int VG = KSV == 2 ? 2 : FC_VG1;
#pragma unroll
          for (int q0 = 0; q0 < kStrip / 14; q0 += VG) {
            if (q0 >= npatch) break;
            uint32_t a[VG][KSV][4];
#pragma unroll
            for (int e2 = 0; e2 < VG; ++e2)
#pragma unroll
              for (int kk = 0; kk < KSV; ++kk) {
                const uint32_t co = (e * SW + 14 * (q0 + e2)) * 4;
                FC_CHK(rb[kk][0] + co >= ring_s && rb[kk][0] + co + 8 <= ring_s + p.TRW * RS * 4 &&
                           rb[kk][1] + co >= ring_s && rb[kk][1] + co + 8 <= ring_s + p.TRW * RS * 4,
                       "V ring read outside the ring");
                const uint2 lo = lds64(rb[kk][0] + co);  // columns 2g, 2g+1; rows k 4t..4t+3
                const uint2 hi = lds64(rb[kk][1] + co);  // k + 16
                a[e2][kk][0] = lo.x;
                a[e2][kk][1] = lo.y;
                a[e2][kk][2] = hi.x;
                a[e2][kk][3] = hi.y;
              }
            int d2[VG][4], d1[VG][4], d0[VG][4];
#pragma unroll
            for (int e2 = 0; e2 < VG; ++e2) fir_mma_planes<KSV>(d2[e2], d1[e2], d0[e2], a[e2], vb);
#pragma unroll
            for (int e2 = 0; e2 < VG; ++e2) {
              const int q = q0 + e2;
              if (q >= npatch) break;
              // d0,d1: column 2g, rows j0, j1; d2,d3: column 2g+1
              int sv[4];
              uint32_t o[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                sv[i] = combine_planes(d2[e2][i], d1[e2][i], d0[e2][i]);  // S = 2^21 + sum T*iv (exact)
                if constexpr (TOK == FC_TOKENS_U8) {
                  o[i] = static_cast<uint32_t>(add_min_relu(sv[i], 0, (1 << 30) - 1)) >> 22;  // the u8 code (NEXT-1)
                } else {  // LUT[clip8(S)] = extended table at floor(S / 2^22) (arithmetic shift)
                  FC_CHK((sv[i] >> 22) >= -kLutLo && (sv[i] >> 22) < 256 + kLutLo,  // every lane: any u8 input stays inside
                         "V value outside the extended normalisation table");
                  o[i] = lds32(lutc + (static_cast<uint32_t>(sv[i] >> 20) & ~3u));
                }
              }
              if constexpr (COLS) {  // NEXT-1: column blocks [W][rows][C] (the paper's last-dimension split)
                const long long rq = static_cast<long long>(r.pair) * static_cast<long long>(pair_rows) +
                                     (static_cast<long long>(hb_) * p.gw2 + X0 / 28) * 4 + (q >> 1) * 4 + (q & 1);
#pragma unroll
                for (int i = 0; i < 4; ++i) {  // o[i]: (j0, 2g) (j1, 2g) (j0, 2g+1) (j1, 2g+1)
                  const int j = (i & 1) ? j1 : j0;
                  const long long rl = rq + (j / 14) * 2;
                  const uint32_t col = (c * 2 + f) * 196 + (j % 14) * 14 + 2 * g + (i >> 1);
                  const uint32_t b = __umulhi(col, p.cs_magic);
                  float* a = static_cast<float*>(p.tokens) + b * p.cs_bstride + rl * p.cs_C + (col - b * p.cs_C);
                  st_cs_pred(a, o[i], ((i & 1) ? jok1 : jok0) && xok);
                }
              } else {
              if constexpr (PAGED) {
                TokT* pb = static_cast<TokT*>(p.tokens) + (c * 2 + f) * 196 + 2 * g;
                st_cs_pred2(pb + static_cast<size_t>(prow[0][q]) * kCols + (j0 % 14) * 14, o[0], o[2], jok0 && xok);
                st_cs_pred2(pb + static_cast<size_t>(prow[1][q]) * kCols + (j1 % 14) * 14, o[1], o[3], jok1 && xok);
              } else {
                TokT* op = tp + (q >> 1) * 4 * kCols + (q & 1) * kCols;  // wb += q/2, wm = q&1
                FC_CHK(p.tokj != nullptr ||
                           ((!(jok0 && xok) || (op >= static_cast<TokT*>(p.tokens) &&
                                                op + 2 <= static_cast<TokT*>(p.tokens) + static_cast<size_t>(p.npairs) * pair_rows * kCols)) &&
                            (!(jok1 && xok) || (op + djo >= static_cast<TokT*>(p.tokens) &&
                                                op + djo + 2 <= static_cast<TokT*>(p.tokens) + static_cast<size_t>(p.npairs) * pair_rows * kCols))),
                       "token store outside the launch's rows");
                st_cs_pred2(op, o[0], o[2], jok0 && xok);        // row j0: columns 2g, 2g+1
                st_cs_pred2(op + djo, o[1], o[3], jok1 && xok);  // row j1
              }
              }
              if (DBG && p.dbg_rs != nullptr) {
                const size_t fi = static_cast<size_t>(p.frame_base + 2 * r.pair + f);
                for (int ee = 0; ee < 4; ++ee) {
                  const int x = X0 + 14 * q + 2 * g + ((ee >= 2) ? 1 : 0), j = (ee & 1) ? j1 : j0;
                  if (xok && x < p.W2 && j < 28)
                    p.dbg_rs[((fi * p.H2 + yo0 + j) * p.W2 + x) * 3 + c] =
                        static_cast<uint32_t>(add_min_relu(sv[ee], 0, (1 << 30) - 1)) >> 22;
                }
              }
            }
          }
        }
      }
#if FC_BAND_BAR
      bar_sync(1, kComputeThreads);  // ring may be overwritten by the next chunks
#endif
      // (no barrier here: the V pass only reads shared memory, and the next
      // ring writes -- the H pass of the next chunk -- come after that chunk's
      // colour->H barrier, which every warp reaches only after its V pass; a
      // warp done early starts converting the next chunk meanwhile)
    }
  }
  if (p.cta_t != nullptr && tid == 0) {
    p.cta_t[3 * blockIdx.x + 1] = globaltimer();
    p.cta_t[3 * blockIdx.x + 2] = smid();
  }
}


// ------------------------------------------------------------ instances
using KernelFn = void (*)(Params);

struct Instance {
  int ksh, ksv;
  KernelFn fn, fn_dbg, fn_bf16, fn_u8;  // fp32 tokens / + parity-test dumps / bf16 tokens / u8 codes
  KernelFn fn_paged, fn_paged_bf16;     // NEXT-2: fp32 / bf16 tokens into a paged pool
  KernelFn fn_i420, fn_i420_dbg;        // I420 surfaces: fp32 tokens / + parity-test dumps
  KernelFn fn_cols;                     // NEXT-1 column-split fp32 output
};

// One translation unit per KSH instantiates its instances (parallel build).
#define FC_INST(A, B)                                                                                  \
  Instance{A, B, fc_fused_kernel<A, B, false, FC_TOKENS_F32>, fc_fused_kernel<A, B, true, FC_TOKENS_F32>, \
           fc_fused_kernel<A, B, false, FC_TOKENS_BF16>, fc_fused_kernel<A, B, false, FC_TOKENS_U8>,   \
           fc_fused_kernel<A, B, false, FC_TOKENS_F32, true>, fc_fused_kernel<A, B, false, FC_TOKENS_BF16, true>, \
           fc_fused_kernel<A, B, false, FC_TOKENS_F32, false, true>, fc_fused_kernel<A, B, true, FC_TOKENS_F32, false, true>, \
           fc_fused_kernel<A, B, false, FC_TOKENS_F32, false, false, true>}
void instances_ksh1(Instance* out);  // out[0..3] = KSV 1..4
void instances_ksh2(Instance* out);
void instances_ksh3(Instance* out);
void instances_ksh4(Instance* out);

}  // namespace fc
