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
#include <string>
#include <vector>

#include "fc_internal.h"

namespace fc {

constexpr int kChunkRows = 16;             // source rows converted per stage-A step
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
  int SWP;            // bytes per source row in the stage-A chunk buffer
  int TR, TRW, TRS;   // ring rows, ring words, column stride in words
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

// Pillow clip8 of the 22-bit fixed-point sum (R4): v>=2^30 -> 255, v<=0 -> 0.
__device__ __forceinline__ uint32_t clip8(uint32_t s) {
  int q = static_cast<int>(s) >> 22;
  return static_cast<uint32_t>(min(max(q, 0), 255));
}

template <int NW>
__device__ __forceinline__ uint32_t fir_bytes(const uint32_t (&d)[NW], const uint32_t (&w0)[NW],
                                              const uint32_t (&w1)[NW], const uint32_t (&w2)[NW]) {
  uint32_t s0 = 1u << 21, s1 = 0, s2 = 0;  // 2^21: Pillow's rounding half
#pragma unroll
  for (int i = 0; i < NW; ++i) {
    s0 = dp4a_uu(d[i], w0[i], s0);
    s1 = dp4a_uu(d[i], w1[i], s1);
    s2 = dp4a_us(d[i], w2[i], s2);
  }
  return clip8(s0 + (s1 << 8) + (s2 << 16));  // modular int32 == exact (R4 headroom)
}

// Integer BT.601 limited range (R3) on 4 pixels: yw = 4 luma bytes, uvw =
// U0 V0 U1 V1 (the 2 chroma samples shared by pixel pairs).  Output: one word
// of 4 bytes per channel.
//   R = (298Y + 409V - 56992) >> 8, G = (298Y - 100U - 208V + 34784) >> 8,
//   B = (298Y + 516U - 70688) >> 8, each clamped to [0,255]
// (the constants fold C = Y-16, D = U-128, E = V-128 and the +128 rounding).
__device__ __forceinline__ void bt601_4(uint32_t yw, uint32_t uvw, uint32_t& R, uint32_t& G, uint32_t& B) {
  R = G = B = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int U = (uvw >> (16 * h)) & 0xFF, V = (uvw >> (16 * h + 8)) & 0xFF;
    const int cr = 409 * V - 56992;
    const int cg = 34784 - 100 * U - 208 * V;
    const int cb = 516 * U - 70688;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int i = 2 * h + k;
      const int y298 = 298 * static_cast<int>((yw >> (8 * i)) & 0xFF);
      const int r = min(max((y298 + cr) >> 8, 0), 255);
      const int g = min(max((y298 + cg) >> 8, 0), 255);
      const int b = min(max((y298 + cb) >> 8, 0), 255);
      R |= static_cast<uint32_t>(r) << (8 * i);
      G |= static_cast<uint32_t>(g) << (8 * i);
      B |= static_cast<uint32_t>(b) << (8 * i);
    }
  }
}

__device__ __forceinline__ void st_cs_f2(float* p, float a, float b) {
  asm volatile("st.global.cs.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(a), "f"(b) : "memory");
}

template <int NW, int K>
__global__ void __launch_bounds__(56 * K) fc_fused_kernel(const __grid_constant__ Params p) {
  constexpr int SW = 28 * K;   // output columns per strip
  constexpr int NT = 2 * SW;   // threads: one per (frame of the pair, column)
  constexpr int CH = kChunkRows;
  constexpr int VWS = 1 + 3 * NW;  // words per vertical-table row in smem
  constexpr int SWR = SW + 4;      // R row stride: odd word count -> conflict-free

  extern __shared__ __align__(16) uint8_t smem[];
  float* lut = reinterpret_cast<float*>(smem);                       // 768 f32
  uint32_t* tab = reinterpret_cast<uint32_t*>(lut + 768);            // 588
  uint32_t* vws = tab + 588;                                          // 28 * VWS
  uint8_t* rgb = reinterpret_cast<uint8_t*>(vws + 28 * VWS);          // [2][3][CH][SWP]
  uint32_t* ring = reinterpret_cast<uint32_t*>(rgb + 6 * CH * p.SWP); // [2][3][SW][TRS]
  uint8_t* Rb = reinterpret_cast<uint8_t*>(ring + 6 * SW * p.TRS);    // [2][3][28][SWR]

  const int tid = threadIdx.x;
  const int strip = blockIdx.x, pair = blockIdx.y;
  const int X0 = strip * SW;
  const int sw_act = min(SW, p.W2 - X0);
  const int SX0 = __ldg(p.hx + X0) & ~15;
  const int NQ = p.SWP >> 4;

  for (int i = tid; i < 768; i += NT) lut[i] = __ldg(p.lut + i);
  for (int e = tid; e < 588; e += NT) {
    const int col = 2 * e, c = col / 392, tp = (col % 392) / 196, ph = (col % 196) / 14, pw = col % 14;
    tab[e] = static_cast<uint32_t>(((tp * 3 + c) * 28 + ph) * SWR + pw) | (static_cast<uint32_t>(c) << 16);
  }

  // horizontal weights of this thread's output column live in registers
  const int hf = tid / SW, ho = tid - hf * SW;
  const bool hact = ho < sw_act;
  uint32_t hw0[NW], hw1[NW], hw2[NW];
  int hoff = 0;
  if (hact) {
    const uint32_t* w = p.hw + static_cast<size_t>(X0 + ho) * 3 * NW;
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      hw0[i] = __ldg(w + i);
      hw1[i] = __ldg(w + NW + i);
      hw2[i] = __ldg(w + 2 * NW + i);
    }
    hoff = __ldg(p.hx + X0 + ho) - SX0;
  } else {
#pragma unroll
    for (int i = 0; i < NW; ++i) hw0[i] = hw1[i] = hw2[i] = 0;
  }
  const int hsh = (hoff & 3) * 8;
  const int hwo = hoff >> 2;

  const FrameDesc* frs = &p.fr[2 * pair];
  int done = 0;  // source rows [.., done) are in the ring (4-aligned)

  for (int hb = 0; hb < p.gh2; ++hb) {
    const int yo0 = hb * 28;
    const int ylo = __ldg(p.vx + yo0) & ~3;
    const int yend = (__ldg(p.vx + yo0 + 27) + __ldg(p.vcnt + yo0 + 27) + 3) & ~3;
    for (int r0 = max(done, ylo); r0 < yend; r0 += CH) {
      const int rows = min(CH, yend - r0);
      // ---- stage A1: NV12 -> RGB planes (a5), 16 pixels per item
      for (int it = tid; it < 2 * rows * NQ; it += NT) {
        const int q = it % NQ;
        const int rr = (it / NQ) % rows;
        const int f = it / (NQ * rows);
        const int y = r0 + rr;
        const int x = SX0 + 16 * q;
        uint4 Yv = make_uint4(0, 0, 0, 0), UVv = make_uint4(0, 0, 0, 0);
        const FrameDesc fd = frs[f];
        if (y < p.H && x < p.W) {
          Yv = __ldg(reinterpret_cast<const uint4*>(fd.y + static_cast<size_t>(y) * fd.py + x));
          UVv = __ldg(reinterpret_cast<const uint4*>(fd.uv + static_cast<size_t>(y >> 1) * fd.puv + x));
        }
        uint4 Rv, Gv, Bv;
        bt601_4(Yv.x, UVv.x, Rv.x, Gv.x, Bv.x);
        bt601_4(Yv.y, UVv.y, Rv.y, Gv.y, Bv.y);
        bt601_4(Yv.z, UVv.z, Rv.z, Gv.z, Bv.z);
        bt601_4(Yv.w, UVv.w, Rv.w, Gv.w, Bv.w);
        uint8_t* dst = rgb + ((f * 3) * CH + rr) * p.SWP + 16 * q;
        *reinterpret_cast<uint4*>(dst) = Rv;
        *reinterpret_cast<uint4*>(dst + CH * p.SWP) = Gv;
        *reinterpret_cast<uint4*>(dst + 2 * CH * p.SWP) = Bv;
        if (p.dbg_src != nullptr && y < p.H) {
          const uint32_t cw[3][4] = {{Rv.x, Rv.y, Rv.z, Rv.w}, {Gv.x, Gv.y, Gv.z, Gv.w}, {Bv.x, Bv.y, Bv.z, Bv.w}};
          const size_t fi = static_cast<size_t>(p.frame_base + 2 * pair + f);
          for (int i = 0; i < 16 && x + i < p.W; ++i)
            for (int c = 0; c < 3; ++c)
              p.dbg_src[((fi * p.H + y) * p.W + x + i) * 3 + c] = (cw[c][i >> 2] >> (8 * (i & 3))) & 0xFF;
        }
      }
      __syncthreads();
      // ---- stage A2: horizontal pass (a6) into the column-major u8 ring
      if (hact) {
        for (int g = 0; g < (rows >> 2); ++g) {
          const int ringw = ((r0 >> 2) + g) % p.TRW;
#pragma unroll 1
          for (int c = 0; c < 3; ++c) {
            uint32_t word = 0;
#pragma unroll
            for (int rr = 0; rr < 4; ++rr) {
              const uint32_t* src =
                  reinterpret_cast<const uint32_t*>(rgb + ((hf * 3 + c) * CH + 4 * g + rr) * p.SWP) + hwo;
              uint32_t w[NW + 1], d[NW];
#pragma unroll
              for (int i = 0; i <= NW; ++i) w[i] = src[i];
#pragma unroll
              for (int i = 0; i < NW; ++i) d[i] = __funnelshift_r(w[i], w[i + 1], hsh);
              word |= fir_bytes<NW>(d, hw0, hw1, hw2) << (8 * rr);
            }
            ring[((hf * 3 + c) * SW + ho) * p.TRS + ringw] = word;
          }
        }
      }
      __syncthreads();
    }
    done = max(done, yend);

    // ---- vertical tables of this band's 28 output rows -> smem
    for (int i = tid; i < 28 * VWS; i += NT) {
      const int j = i / VWS, k = i - j * VWS;
      const int yo = yo0 + j;
      vws[i] = (k == 0) ? static_cast<uint32_t>(__ldg(p.vx + yo) % p.TR)
                        : __ldg(p.vw + static_cast<size_t>(yo) * 3 * NW + (k - 1));
    }
    __syncthreads();

    // ---- stage B: vertical pass (a7) -> R[f][c][j][x] u8
    // lanes run over output rows j (distinct ring words, conflict-free)
    for (int it = tid; it < 14 * SW; it += NT) {
      const int j = it % 28;
      const int q = (it / 28) % (SW / 4);
      const int f = it / (7 * SW);
      const uint32_t* vj = vws + j * VWS;
      const int ypos = static_cast<int>(vj[0]);
      const int vwo = ypos >> 2, vsh = (ypos & 3) * 8;
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
        const int t = vwo + i;
        widx[i] = t >= p.TRW ? t - p.TRW : t;
      }
#pragma unroll 1
      for (int c = 0; c < 3; ++c) {
        uint32_t outw = 0;
#pragma unroll
        for (int xx = 0; xx < 4; ++xx) {
          const uint32_t* col = ring + ((f * 3 + c) * SW + 4 * q + xx) * p.TRS;
          uint32_t w[NW + 1], d[NW];
#pragma unroll
          for (int i = 0; i <= NW; ++i) w[i] = col[widx[i]];
#pragma unroll
          for (int i = 0; i < NW; ++i) d[i] = __funnelshift_r(w[i], w[i + 1], vsh);
          outw |= fir_bytes<NW>(d, v0, v1, v2) << (8 * xx);
        }
        *reinterpret_cast<uint32_t*>(Rb + ((f * 3 + c) * 28 + j) * SWR + 4 * q) = outw;
        if (p.dbg_rs != nullptr) {
          const size_t fi = static_cast<size_t>(p.frame_base + 2 * pair + f);
          for (int xx = 0; xx < 4; ++xx) {
            const int x = X0 + 4 * q + xx;
            if (x < p.W2)
              p.dbg_rs[((fi * p.H2 + yo0 + j) * p.W2 + x) * 3 + c] = (outw >> (8 * xx)) & 0xFF;
          }
        }
      }
    }
    __syncthreads();

    // ---- stage C: normalise (a8) + patchify (a9), coalesced float2 stores
    {
      const int kact = min(K, p.gw2 - strip * K);
      const int nrows = 4 * kact;
      const size_t row0 = (static_cast<size_t>(pair) * p.gh2 * p.gw2 + static_cast<size_t>(hb) * p.gw2 +
                           static_cast<size_t>(strip) * K) * 4;
      float* out = p.tokens + row0 * kCols;
      for (int it = tid; it < nrows * 588; it += NT) {
        const int r = it / 588, e = it - r * 588;
        const uint32_t te = tab[e];
        const int wbl = r >> 2, hm = (r >> 1) & 1, wm = r & 1;
        const int roff = static_cast<int>(te & 0xFFFF) + 14 * hm * SWR + 28 * wbl + 14 * wm;
        const uint32_t v2 = *reinterpret_cast<const uint16_t*>(Rb + roff);
        const float* l = lut + (te >> 16) * 256;
        st_cs_f2(out + static_cast<size_t>(it) * 2, l[v2 & 0xFF], l[v2 >> 8]);
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

static fc_status device_tables(fc_plan_s* P, int dev, DeviceTables** out) {
  std::lock_guard<std::mutex> lk(P->mu);
  auto it = P->dev.find(dev);
  if (it != P->dev.end()) {
    *out = &it->second;
    return FC_OK;
  }
  const int nw = plan_nw(P);
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
  *out = &(P->dev[dev] = t);
  return FC_OK;
}

struct Geometry {
  int K, nw, SWP, TR, TRW, TRS, nstrips;
  size_t smem;
};

static size_t smem_bytes(int K, int nw, int SWP, int TRS) {
  const int SW = 28 * K;
  return 768 * 4 + 588 * 4 + 28 * (1 + 3 * nw) * 4 + static_cast<size_t>(6) * kChunkRows * SWP +
         static_cast<size_t>(6) * SW * TRS * 4 + static_cast<size_t>(6) * 28 * (SW + 4);
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
  int tr = 4 * (nw + 1);
  for (int hb = 0; hb < P->h2 / 28; ++hb) {
    const int ylo = tv.xmin[hb * 28] & ~3;
    const int yend = (tv.xmin[hb * 28 + 27] + tv.cnt[hb * 28 + 27] + 3) & ~3;
    tr = std::max(tr, yend - ylo);
  }
  tr = (tr + 3) & ~3;
  g->K = K;
  g->nw = nw;
  g->SWP = swp;
  g->TR = tr;
  g->TRW = tr / 4;
  g->TRS = (g->TRW & 1) ? g->TRW : g->TRW + 1;
  g->nstrips = nstrips;
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
    fn<<<grid, 56 * g.K, g.smem, s>>>(prm);
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
  if (!P) return;
  for (auto& kv : P->dev) {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(kv.first);
    DeviceTables& t = kv.second;
    cudaFree(t.hx); cudaFree(t.hcnt); cudaFree(t.hw); cudaFree(t.vx); cudaFree(t.vcnt); cudaFree(t.vw);
    cudaFree(t.lut);
    cudaSetDevice(cur);
  }
  delete P;
}

}  // extern "C"
