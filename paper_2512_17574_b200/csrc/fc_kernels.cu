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
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "fc_device.cuh"
#include "fc_internal.h"

namespace fc {

constexpr int kChunkRows = 16;             // source rows per stage-A chunk
constexpr int kMaxFramesPerLaunch = 1200;  // frame descriptors passed by value

struct FrameDesc {
  const uint8_t* y;
  const uint8_t* uv;
  int32_t py, puv;
};

struct Params {
  int W, H, W2, H2;
  int gh2, gw2;       // merge blocks per column / row
  int nstrips;
  int SWP;            // bytes per source row in the chunk buffers
  int TR, TRW, TRS;   // ring rows, ring words, column stride in words
  int nchunks;        // ceil(H / 16)
  const int32_t* hx;
  const uint32_t* hw;
  const int32_t* vx;
  const int32_t* vcnt;
  const uint32_t* vw;
  const float* lut;
  float* tokens;      // first token row of this launch's first pair
  uint8_t* dbg_src;   // [nframes_total, H, W, 3] or null
  uint8_t* dbg_rs;    // [nframes_total, H2, W2, 3] or null
  int frame_base;     // index of fr[0] within the rank's frame list (debug dumps)
  int nframes;
  FrameDesc fr[kMaxFramesPerLaunch];
};

// Issue the TMA bulk copies of one 16-row chunk (both frames, Y rows + the
// 8 UV rows) into raw buffer `buf`.  Executed by warp 0; lane 0 arms the
// mbarrier with the chunk's byte count first.
__device__ __forceinline__ void issue_chunk(const Params& p, const FrameDesc* frs, int SX0, int k, uint8_t* raw,
                                            uint64_t* bar, int lane) {
  const int r0 = k * kChunkRows;
  const int rows_y = min(kChunkRows, p.H - r0);
  const int rows_uv = min(kChunkRows / 2, (p.H >> 1) - (r0 >> 1));
  if (lane == 0) {
    uint32_t bytes = 0;
#pragma unroll
    for (int f = 0; f < 2; ++f) {
      const int fy = max(min(p.SWP, frs[f].py - SX0), 0), fuv = max(min(p.SWP, frs[f].puv - SX0), 0);
      bytes += rows_y * fy + rows_uv * fuv;
    }
    mbar_arrive_expect_tx(bar, bytes);
  }
  __syncwarp();
  // 2 frames x 24 rows = 48 copies spread over the warp
  for (int i = lane; i < 48; i += 32) {
    const int f = i / 24, rr = i % 24;
    const FrameDesc fd = frs[f];
    uint8_t* dst = raw + (f * 24 + rr) * p.SWP;
    if (rr < kChunkRows) {
      const int fy = max(min(p.SWP, fd.py - SX0), 0);
      if (rr < rows_y && fy > 0)
        bulk_g2s(dst, fd.y + static_cast<size_t>(r0 + rr) * fd.py + SX0, fy, bar);
    } else {
      const int u = rr - kChunkRows;
      const int fuv = max(min(p.SWP, fd.puv - SX0), 0);
      if (u < rows_uv && fuv > 0)
        bulk_g2s(dst, fd.uv + static_cast<size_t>((r0 >> 1) + u) * fd.puv + SX0, fuv, bar);
    }
  }
}

template <int NW, int K>
__global__ void __launch_bounds__(84 * K, 2) fc_fused_kernel(const __grid_constant__ Params p) {
  constexpr int SW = 28 * K;       // output columns per strip
  constexpr int NT = 3 * SW;       // threads: one per (channel, column) for the H pass
  constexpr int CH = kChunkRows;
  constexpr int VWS = 1 + 3 * NW;  // words per vertical-table row in smem

  extern __shared__ __align__(1024) uint8_t smem[];
  float* lut = reinterpret_cast<float*>(smem);                        // 3 x 256 f32, 1 KB aligned
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 3072);          // 2 mbarriers
  uint32_t* vws = reinterpret_cast<uint32_t*>(smem + 3072 + 16);      // 28 * VWS
  uint8_t* raw = smem + 3072 + 16 + ((28 * VWS * 4 + 15) & ~15);      // [2 buf][2 f][24 rows][SWP]
  uint8_t* rgb = raw + 2 * 48 * p.SWP;                                // [2 f][3 c][16 rows][SWP]
  uint32_t* ring = reinterpret_cast<uint32_t*>(rgb + 6 * CH * p.SWP); // [2 f][3 c][SW][TRS]

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int strip = blockIdx.x, pair = blockIdx.y;
  const int X0 = strip * SW;
  const int sw_act = min(SW, p.W2 - X0);
  const int SX0 = __ldg(p.hx + X0) & ~15;
  const int NQ = p.SWP >> 4;
  const FrameDesc* frs = &p.fr[2 * pair];

  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  for (int i = tid; i < 768; i += NT) lut[i] = __ldg(p.lut + i);
  __syncthreads();
  if (warp == 0) issue_chunk(p, frs, SX0, 0, raw, &bars[0], lane);

  // H pass: thread = (channel hc, column ho) for both frames; weights in registers
  const int hc = tid / SW, ho = tid - hc * SW;
  const bool hact = ho < sw_act;
  uint32_t hw0[NW], hw1[NW], hw2[NW];
  int hoff = 0;
  {
    const int oo = X0 + min(ho, sw_act - 1);
    const uint32_t* w = p.hw + static_cast<size_t>(oo) * 3 * NW;
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      hw0[i] = __ldg(w + i);
      hw1[i] = __ldg(w + NW + i);
      hw2[i] = __ldg(w + 2 * NW + i);
    }
    hoff = __ldg(p.hx + oo) - SX0;
  }
  const int hsh = (hoff & 3) * 8;
  const uint8_t* hsrc0 = rgb + (hc * CH) * p.SWP + (hoff & ~3);     // frame 0, row 0
  const uint8_t* hsrc1 = hsrc0 + 3 * CH * p.SWP;                      // frame 1
  uint32_t* hdst0 = ring + (hc * SW + ho) * p.TRS;
  uint32_t* hdst1 = hdst0 + 3 * SW * p.TRS;

  // V pass: thread = (channel vc, column pair vxp, half of the band vjh), both frames
  const int vc = tid / SW, vrem = tid - vc * SW;
  const int vxp = vrem % (SW / 2), vjh = vrem / (SW / 2);
  const int vx = 2 * vxp;
  const bool vact = vx < sw_act;
  const uint32_t* vcol00 = ring + (vc * SW + vx) * p.TRS;   // frame 0, column vx
  const uint32_t* vcol01 = vcol00 + p.TRS;                  // frame 0, column vx+1
  const uint32_t* vcol10 = vcol00 + 3 * SW * p.TRS;         // frame 1
  const uint32_t* vcol11 = vcol10 + p.TRS;
  const uint32_t lutb = smem_u32(lut + vc * 256);
  // token addressing of this thread's columns (R6): x = 28 wb + 14 wm + pw
  const int gx = X0 + vx;
  const int vwb = gx / 28, vwm = (gx / 14) & 1, vpw = gx % 14;

  int next_k = 0;
  for (int hb = 0; hb < p.gh2; ++hb) {
    const int yo0 = hb * 28;
    const int yend = __ldg(p.vx + yo0 + 27) + __ldg(p.vcnt + yo0 + 27);
    const int kneed = min(p.nchunks, (yend + CH - 1) / CH);
    for (; next_k < kneed; ++next_k) {
      const int k = next_k, buf = k & 1;
      uint8_t* rawb = raw + buf * 48 * p.SWP;
      if (warp == 0 && k + 1 < p.nchunks) {
        fence_proxy_async();
        issue_chunk(p, frs, SX0, k + 1, raw + (buf ^ 1) * 48 * p.SWP, &bars[buf ^ 1], lane);
      }
      mbar_wait(&bars[buf], (k >> 1) & 1);
      // ---- a5: NV12 -> RGB planes, 16 pixels per item
      const int r0 = k * CH;
      for (int it = tid; it < 2 * CH * NQ; it += NT) {
        const int q = it % NQ;
        const int rr = (it / NQ) % CH;
        const int f = it / (NQ * CH);
        const uint4 Yv = *reinterpret_cast<const uint4*>(rawb + (f * 24 + rr) * p.SWP + 16 * q);
        const uint4 UVv = *reinterpret_cast<const uint4*>(rawb + (f * 24 + CH + (rr >> 1)) * p.SWP + 16 * q);
        uint4 Rv, Gv, Bv;
        bt601_4(Yv.x, UVv.x, Rv.x, Gv.x, Bv.x);
        bt601_4(Yv.y, UVv.y, Rv.y, Gv.y, Bv.y);
        bt601_4(Yv.z, UVv.z, Rv.z, Gv.z, Bv.z);
        bt601_4(Yv.w, UVv.w, Rv.w, Gv.w, Bv.w);
        uint8_t* dst = rgb + ((f * 3) * CH + rr) * p.SWP + 16 * q;
        *reinterpret_cast<uint4*>(dst) = Rv;
        *reinterpret_cast<uint4*>(dst + CH * p.SWP) = Gv;
        *reinterpret_cast<uint4*>(dst + 2 * CH * p.SWP) = Bv;
        if (p.dbg_src != nullptr) {
          const int y = r0 + rr, x = SX0 + 16 * q;
          if (y < p.H) {
            const uint32_t cw[3][4] = {{Rv.x, Rv.y, Rv.z, Rv.w}, {Gv.x, Gv.y, Gv.z, Gv.w}, {Bv.x, Bv.y, Bv.z, Bv.w}};
            const size_t fi = static_cast<size_t>(p.frame_base + 2 * pair + f);
            for (int i = 0; i < 16 && x + i < p.W; ++i)
              for (int c = 0; c < 3; ++c)
                p.dbg_src[((fi * p.H + y) * p.W + x + i) * 3 + c] = (cw[c][i >> 2] >> (8 * (i & 3))) & 0xFF;
          }
        }
      }
      __syncthreads();
      // ---- a6: horizontal pass -> ring (4 rows packed per word, column-major)
      if (hact) {
        const int wbase = ((r0 >> 2) % p.TRW);
#pragma unroll 1
        for (int g = 0; g < CH / 4; ++g) {
          int qa[4], qb[4];
#pragma unroll
          for (int rr = 0; rr < 4; ++rr) {
            const int row = 4 * g + rr;
            const uint32_t* s0 = reinterpret_cast<const uint32_t*>(hsrc0 + row * p.SWP);
            const uint32_t* s1 = reinterpret_cast<const uint32_t*>(hsrc1 + row * p.SWP);
            uint32_t a[NW + 1], b[NW + 1], da[NW], db[NW];
#pragma unroll
            for (int i = 0; i <= NW; ++i) {
              a[i] = s0[i];
              b[i] = s1[i];
            }
#pragma unroll
            for (int i = 0; i < NW; ++i) {
              da[i] = __funnelshift_r(a[i], a[i + 1], hsh);
              db[i] = __funnelshift_r(b[i], b[i + 1], hsh);
            }
            qa[rr] = fir_sum<NW>(da, hw0, hw1, hw2) >> 22;  // clip8 = saturating pack below
            qb[rr] = fir_sum<NW>(db, hw0, hw1, hw2) >> 22;
          }
          const uint32_t word0 = pack_sat_u8(qa[1], qa[0], pack_sat_u8(qa[3], qa[2], 0));
          const uint32_t word1 = pack_sat_u8(qb[1], qb[0], pack_sat_u8(qb[3], qb[2], 0));
          int w = wbase + g;
          if (w >= p.TRW) w -= p.TRW;
          hdst0[w] = word0;
          hdst1[w] = word1;
        }
      }
      __syncthreads();
    }
    // ---- vertical tables of this band's 28 output rows -> smem
    for (int i = tid; i < 28 * VWS; i += NT) {
      const int j = i / VWS, kk = i - j * VWS;
      const int yo = yo0 + j;
      vws[i] = (kk == 0) ? static_cast<uint32_t>(__ldg(p.vx + yo) % p.TR)
                         : __ldg(p.vw + static_cast<size_t>(yo) * 3 * NW + (kk - 1));
    }
    __syncthreads();
    // ---- a7 + a8 + a9: vertical pass, normalise, patchify (float2 stores)
    if (vact) {
      const size_t trow = (static_cast<size_t>(pair) * p.gh2 + hb) * p.gw2 * 4 + vwb * 4 + vjh * 2 + vwm;
      float* out0 = p.tokens + trow * kCols + (vc * 2 + 0) * 196 + vpw;
      float* out1 = out0 + 196;
#pragma unroll 1
      for (int jj = 0; jj < 14; ++jj) {
        const int j = vjh * 14 + jj;
        const uint32_t* vj = vws + j * VWS;
        const int ypos = static_cast<int>(vj[0]);
        const int vsh = (ypos & 3) * 8;
        uint32_t v0[NW], v1[NW], v2[NW];
#pragma unroll
        for (int i = 0; i < NW; ++i) {
          v0[i] = vj[1 + i];
          v1[i] = vj[1 + NW + i];
          v2[i] = vj[1 + 2 * NW + i];
        }
        int widx[NW + 1];
#pragma unroll
        for (int i = 0; i <= NW; ++i) {
          const int t = (ypos >> 2) + i;
          widx[i] = t >= p.TRW ? t - p.TRW : t;
        }
        uint32_t a0[NW + 1], a1[NW + 1], b0[NW + 1], b1[NW + 1];
#pragma unroll
        for (int i = 0; i <= NW; ++i) {
          a0[i] = vcol00[widx[i]];
          a1[i] = vcol01[widx[i]];
          b0[i] = vcol10[widx[i]];
          b1[i] = vcol11[widx[i]];
        }
        uint32_t da0[NW], da1[NW], db0[NW], db1[NW];
#pragma unroll
        for (int i = 0; i < NW; ++i) {
          da0[i] = __funnelshift_r(a0[i], a0[i + 1], vsh);
          da1[i] = __funnelshift_r(a1[i], a1[i + 1], vsh);
          db0[i] = __funnelshift_r(b0[i], b0[i + 1], vsh);
          db1[i] = __funnelshift_r(b1[i], b1[i + 1], vsh);
        }
        // clip8 then table index: clamp S to [0, 2^30-1], byte = S >> 22
        const uint32_t s00 = static_cast<uint32_t>(add_min_relu(fir_sum<NW>(da0, v0, v1, v2), 0, (1 << 30) - 1));
        const uint32_t s01 = static_cast<uint32_t>(add_min_relu(fir_sum<NW>(da1, v0, v1, v2), 0, (1 << 30) - 1));
        const uint32_t s10 = static_cast<uint32_t>(add_min_relu(fir_sum<NW>(db0, v0, v1, v2), 0, (1 << 30) - 1));
        const uint32_t s11 = static_cast<uint32_t>(add_min_relu(fir_sum<NW>(db1, v0, v1, v2), 0, (1 << 30) - 1));
        float o00, o01, o10, o11;
        asm("ld.shared.f32 %0, [%1];" : "=f"(o00) : "r"(((s00 >> 20) & 0x3FCu) + lutb));
        asm("ld.shared.f32 %0, [%1];" : "=f"(o01) : "r"(((s01 >> 20) & 0x3FCu) + lutb));
        asm("ld.shared.f32 %0, [%1];" : "=f"(o10) : "r"(((s10 >> 20) & 0x3FCu) + lutb));
        asm("ld.shared.f32 %0, [%1];" : "=f"(o11) : "r"(((s11 >> 20) & 0x3FCu) + lutb));
        st_cs_f2(out0 + jj * 14, o00, o01);
        st_cs_f2(out1 + jj * 14, o10, o11);
        if (p.dbg_rs != nullptr) {
          const size_t fi0 = static_cast<size_t>(p.frame_base + 2 * pair);
          const int yo = yo0 + j;
          uint8_t* d0 = p.dbg_rs + ((fi0 * p.H2 + yo) * p.W2 + gx) * 3 + vc;
          uint8_t* d1 = d0 + static_cast<size_t>(p.H2) * p.W2 * 3;
          d0[0] = s00 >> 22;
          d0[3] = s01 >> 22;
          d1[0] = s10 >> 22;
          d1[3] = s11 >> 22;
        }
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ host side
static const int kNW[] = {1, 2, 3, 4, 6, 8, 12, 16};

static int pick_nw(int words) {
  for (int w : kNW)
    if (w >= words) return w;
  return -1;
}

using KernelFn = void (*)(Params);

template <int NW, int K>
static KernelFn kfn() {
  return fc_fused_kernel<NW, K>;
}

static KernelFn select_kernel(int nw, int K) {
#define FC_CASE(NWV)                                  \
  case NWV:                                           \
    return K == 4 ? kfn<NWV, 4>() : kfn<NWV, 2>();
  switch (nw) {
    FC_CASE(1)
    FC_CASE(2)
    FC_CASE(3)
    FC_CASE(4)
    FC_CASE(6)
    FC_CASE(8)
    FC_CASE(12)
    FC_CASE(16)
  }
#undef FC_CASE
  return nullptr;
}

static fc_status cuda_fail(cudaError_t e, const char* what) {
  return fail(FC_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Re-pack an axis table's byte planes to the kernel's word count.
static std::vector<uint32_t> planes_for(const AxisTable& t, int nw) {
  std::vector<uint32_t> out(static_cast<size_t>(t.out) * 3 * nw, 0u);
  for (int o = 0; o < t.out; ++o)
    for (int pl = 0; pl < 3; ++pl)
      for (int i = 0; i < t.words; ++i)
        out[(static_cast<size_t>(o) * 3 + pl) * nw + i] = t.planes[(static_cast<size_t>(o) * 3 + pl) * t.words + i];
  return out;
}

template <typename T>
static cudaError_t upload(T** dst, const std::vector<T>& v) {
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(dst), std::max<size_t>(v.size(), 1) * sizeof(T));
  if (e != cudaSuccess) return e;
  return cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
}

static int plan_nw(const fc_plan_s* P) { return pick_nw(std::max(P->th.words, P->tv.words)); }

// Process-wide cache of uploaded tables, keyed by everything the tables are
// a function of (device, W->W', H->H', packing width, normalisation).  Plans
// of equally shaped requests share one upload, so fc_plan + fc_preprocess
// never touch the device synchronously after the first request of a shape.
struct TableKey {
  int dev, w, w2, h, h2, nw;
  uint32_t lut_bits[768];
  bool operator<(const TableKey& o) const {
    return std::memcmp(this, &o, sizeof(TableKey)) < 0;
  }
};

static std::mutex g_tables_mu;
static std::map<TableKey, DeviceTables>* g_tables = new std::map<TableKey, DeviceTables>();  // never freed

static fc_status device_tables(fc_plan_s* P, int dev, DeviceTables** out) {
  std::lock_guard<std::mutex> lk(P->mu);
  auto it = P->dev.find(dev);
  if (it != P->dev.end()) {
    *out = &it->second;
    return FC_OK;
  }
  const int nw = plan_nw(P);
  TableKey key;
  std::memset(&key, 0, sizeof(key));
  key.dev = dev;
  key.w = P->th.in;
  key.w2 = P->th.out;
  key.h = P->tv.in;
  key.h2 = P->tv.out;
  key.nw = nw;
  std::memcpy(key.lut_bits, P->lut.data(), sizeof(key.lut_bits));
  std::lock_guard<std::mutex> gk(g_tables_mu);
  auto git = g_tables->find(key);
  if (git != g_tables->end()) {
    *out = &(P->dev[dev] = git->second);
    return FC_OK;
  }
  DeviceTables t;
  cudaError_t e = cudaSuccess;
  if (e == cudaSuccess) e = upload(&t.hx, P->th.xmin);
  if (e == cudaSuccess) e = upload(&t.hcnt, P->th.cnt);
  if (e == cudaSuccess) e = upload(&t.hw, planes_for(P->th, nw));
  if (e == cudaSuccess) e = upload(&t.vx, P->tv.xmin);
  if (e == cudaSuccess) e = upload(&t.vcnt, P->tv.cnt);
  if (e == cudaSuccess) e = upload(&t.vw, planes_for(P->tv, nw));
  if (e == cudaSuccess) e = upload(&t.lut, P->lut);
  if (e != cudaSuccess) {
    cudaFree(t.hx); cudaFree(t.hcnt); cudaFree(t.hw); cudaFree(t.vx); cudaFree(t.vcnt); cudaFree(t.vw);
    cudaFree(t.lut);
    return e == cudaErrorMemoryAllocation ? fail(FC_ERR_OOM, "table upload: out of device memory")
                                          : cuda_fail(e, "table upload");
  }
  (*g_tables)[key] = t;
  *out = &(P->dev[dev] = t);
  return FC_OK;
}

struct Geometry {
  int K, nw, SWP, TR, TRW, TRS, nstrips, nchunks;
  size_t smem;
};

static size_t smem_bytes(int K, int nw, int SWP, int TRS) {
  const int SW = 28 * K;
  return 3072 + 16 + ((28 * (1 + 3 * nw) * 4 + 15) & ~15) + static_cast<size_t>(2) * 48 * SWP +
         static_cast<size_t>(6) * kChunkRows * SWP + static_cast<size_t>(6) * SW * TRS * 4;
}

static bool geometry(const fc_plan_s* P, int K, Geometry* g) {
  const int SW = 28 * K;
  const int nw = plan_nw(P);
  if (nw < 0) return false;
  const auto& th = P->th;
  const auto& tv = P->tv;
  int swp = 16;
  const int nstrips = (P->w2 + SW - 1) / SW;
  for (int s = 0; s < nstrips; ++s) {
    const int X0 = s * SW, X1 = std::min(X0 + SW, P->w2);
    const int SX0 = th.xmin[X0] & ~15;
    int need = 0;
    for (int o = X0; o < X1; ++o) {
      const int off = th.xmin[o] - SX0;
      need = std::max(need, (off & ~3) + 4 * (nw + 1));
      need = std::max(need, th.xmin[o] + th.cnt[o] - SX0);
    }
    swp = std::max(swp, (need + 15) & ~15);
  }
  // ring: after the chunks a band needs (16-row granularity) the ring must
  // still hold the band's first source row
  int tr = 4 * (nw + 1);
  int kmax = 0;
  for (int hb = 0; hb < P->h2 / 28; ++hb) {
    const int ylo = tv.xmin[hb * 28] & ~3;
    const int yend = tv.xmin[hb * 28 + 27] + tv.cnt[hb * 28 + 27];
    const int kneed = (yend + kChunkRows - 1) / kChunkRows;
    tr = std::max(tr, kneed * kChunkRows - ylo);
    kmax = std::max(kmax, kneed);
  }
  tr = (tr + 3) & ~3;
  g->K = K;
  g->nw = nw;
  g->SWP = swp;
  g->TR = tr;
  g->TRW = tr / 4;
  g->TRS = (g->TRW & 1) ? g->TRW : g->TRW + 1;
  g->nstrips = nstrips;
  g->nchunks = std::min(kmax, (P->meta.height + kChunkRows - 1) / kChunkRows);
  g->smem = smem_bytes(K, nw, swp, g->TRS);
  return true;
}

static fc_status choose_geometry(const fc_plan_s* P, int max_smem, Geometry* g) {
  for (int K : {4, 2}) {
    if (!geometry(P, K, g)) return fail(FC_ERR_UNSUPPORTED, "resize filter too wide");
    // prefer K=4 only when two CTAs fit per SM
    if (K == 4 && g->smem * 2 > static_cast<size_t>(max_smem)) continue;
    if (g->smem <= static_cast<size_t>(max_smem)) return FC_OK;
  }
  return fail(FC_ERR_UNSUPPORTED, "working set exceeds shared memory (frame too wide for one strip)");
}

static fc_status preprocess_impl(const fc_plan_t* Pc, int32_t rank, const fc_nv12_surface* surfaces,
                                 int64_t num_surfaces, float* tokens, int64_t grid_thw[3], void* stream,
                                 uint8_t* dbg_src, uint8_t* dbg_rs) {
  if (!Pc) return fail(FC_ERR_INVALID_ARG, "plan is NULL");
  fc_plan_s* P = const_cast<fc_plan_s*>(Pc);
  if (rank < 0 || rank >= P->world) return fail(FC_ERR_RANK, "rank outside [0, world_size)");
  const fc_rank_plan& rp = P->ranks[rank].p;
  if (grid_thw) {
    grid_thw[0] = P->gt;
    grid_thw[1] = P->gh;
    grid_thw[2] = P->gw;
  }
  if (rp.row_end == rp.row_begin) return FC_OK;
  if (!surfaces || !tokens) return fail(FC_ERR_INVALID_ARG, "surfaces/tokens is NULL");
  // the rank's frame list: its sampled frames, then pad copies of the last
  std::vector<int64_t> frames;
  for (int64_t i = 0; i < rp.sampled_count; ++i) frames.push_back(P->sampled[rp.sampled_begin + i]);
  for (int64_t i = 0; i < rp.pad_frames; ++i) frames.push_back(frames.back());
  const int W = P->meta.width, H = P->meta.height;
  for (int64_t f : frames) {
    if (f >= num_surfaces) return fail(FC_ERR_MISSING_SURFACE, "surface array too short for frame " + std::to_string(f));
    const fc_nv12_surface& s = surfaces[f];
    if (!s.y || !s.uv) return fail(FC_ERR_MISSING_SURFACE, "NULL surface for frame " + std::to_string(f));
    if ((reinterpret_cast<uintptr_t>(s.y) & 15) || (reinterpret_cast<uintptr_t>(s.uv) & 15))
      return fail(FC_ERR_UNSUPPORTED, "surface planes must be 16-byte aligned");
    if ((s.pitch_y & 15) || (s.pitch_uv & 15) || s.pitch_y < W || s.pitch_uv < W || s.pitch_y > INT32_MAX ||
        s.pitch_uv > INT32_MAX)
      return fail(FC_ERR_UNSUPPORTED, "pitches must be multiples of 16 and >= width");
  }
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  int major = 0, max_smem = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (major != 10) return fail(FC_ERR_CUDA, "fc kernels are built for sm_100a only (no CPU/other-arch fallback)");
  Geometry g;
  fc_status st = choose_geometry(P, max_smem, &g);
  if (st != FC_OK) return st;
  DeviceTables* dt = nullptr;
  st = device_tables(P, dev, &dt);
  if (st != FC_OK) return st;
  KernelFn fn = select_kernel(g.nw, g.K);
  if (!fn) return fail(FC_ERR_UNSUPPORTED, "no kernel instance for this filter width");
  e = cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(g.smem));
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");

  static thread_local Params prm;  // ~30 KB: keep it off the stack
  std::memset(&prm, 0, offsetof(Params, fr));
  prm.W = W;
  prm.H = H;
  prm.W2 = P->w2;
  prm.H2 = P->h2;
  prm.gh2 = static_cast<int>(P->gh / 2);
  prm.gw2 = static_cast<int>(P->gw / 2);
  prm.nstrips = g.nstrips;
  prm.SWP = g.SWP;
  prm.TR = g.TR;
  prm.TRW = g.TRW;
  prm.TRS = g.TRS;
  prm.nchunks = g.nchunks;
  prm.hx = dt->hx;
  prm.hw = dt->hw;
  prm.vx = dt->vx;
  prm.vcnt = dt->vcnt;
  prm.vw = dt->vw;
  prm.lut = dt->lut;
  prm.dbg_src = dbg_src;
  prm.dbg_rs = dbg_rs;
  const int64_t nf = static_cast<int64_t>(frames.size());
  const int64_t rows_per_pair = P->gh * P->gw;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  for (int64_t f0 = 0; f0 < nf; f0 += kMaxFramesPerLaunch) {
    const int64_t cnt = std::min<int64_t>(kMaxFramesPerLaunch, nf - f0);
    prm.frame_base = static_cast<int>(f0);
    prm.nframes = static_cast<int>(cnt);
    prm.tokens = tokens + (f0 / 2) * rows_per_pair * kCols;
    for (int64_t i = 0; i < cnt; ++i) {
      const fc_nv12_surface& sf = surfaces[frames[f0 + i]];
      prm.fr[i] = FrameDesc{sf.y, sf.uv, static_cast<int32_t>(sf.pitch_y), static_cast<int32_t>(sf.pitch_uv)};
    }
    dim3 grid(g.nstrips, static_cast<unsigned>(cnt / 2));
    fn<<<grid, 84 * g.K, g.smem, s>>>(prm);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  }
  return FC_OK;
}

}  // namespace fc

using namespace fc;

extern "C" {

fc_status fc_preprocess(const fc_plan_t* plan, int32_t rank, const fc_nv12_surface* surfaces,
                        int64_t num_surfaces, float* tokens, int64_t grid_thw[3], void* stream) {
  return preprocess_impl(plan, rank, surfaces, num_surfaces, tokens, grid_thw, stream, nullptr, nullptr);
}

fc_status fc_preprocess_debug(const fc_plan_t* plan, int32_t rank, const fc_nv12_surface* surfaces,
                              int64_t num_surfaces, float* tokens, int64_t grid_thw[3], void* stream,
                              uint8_t* rgb_src, uint8_t* rgb_resized) {
  return preprocess_impl(plan, rank, surfaces, num_surfaces, tokens, grid_thw, stream, rgb_src, rgb_resized);
}

fc_status fc_preprocess_batch(const fc_plan_t* const* plans, const int32_t* ranks, int32_t count,
                              const fc_nv12_surface* const* surfaces, const int64_t* num_surfaces,
                              float* const* tokens, void* stream) {
  if (count < 0 || (count > 0 && (!plans || !ranks || !surfaces || !num_surfaces || !tokens)))
    return fail(FC_ERR_INVALID_ARG, "batch arguments");
  // v0: one launch per job (a single work-list launch is on the roadmap)
  for (int32_t i = 0; i < count; ++i) {
    fc_status st = preprocess_impl(plans[i], ranks[i], surfaces[i], num_surfaces[i], tokens[i], nullptr, stream,
                                   nullptr, nullptr);
    if (st != FC_OK) return st;
  }
  return FC_OK;
}

void fc_plan_destroy(fc_plan_t* P) {
  // device tables belong to the process-wide cache (shared by equal shapes)
  delete P;
}

}  // extern "C"
