// fc_tc.cu -- host side of the tcgen05 kernel (fc_tc.cuh): weight-digit
// tables in the UMMA core-matrix layouts, the shared-memory plan, launch.
//
// Tables (per device, cached process-wide per (W->W', H->H', normalisation)):
//   hB   [nstrips][192 x KH]  H-pass B operand: n = digit*64 + output column
//        of the strip, k = source column - SX0; K-major core matrices
//        (8 rows x 16 B, K-chunk stride 128 B, 8-row stride KH/16*128 B).
//        Plane 2 carries +32 at k = KH-1, the A column the kernel sets to 1:
//        Pillow's rounding term 2^21 = 32 * 2^16 (R4).
//   vB   [gh2][2][48 x KV]    V-pass B operand per half band: n = digit*16 +
//        output row, k = source row - ys8.
//   vys  [gh2][2]  8-aligned first source row of each half band's window.
//   vcl  [gh2]     last 16-row chunk with a nonzero weight of the band.
//   lut2 [3][704]  doubled normalisation table (R5): entry a + 97 is
//        LUT[clip8(floor((a + 1) / 2))] for a = floor(S / 2^21).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "fc_launch.h"
#include "fc_tc.cuh"

namespace fc {
namespace tc {

void tc_kernels(TcKernelFn* prod, TcKernelFn* dbg, TcKernelFn* prof) {
  *prod = fc_tc_kernel<false>;
  *dbg = fc_tc_kernel<true>;
  *prof = fc_tc_kernel<false, true>;
}

namespace {

struct TcTables {
  TcTables() = default;
  TcTables(const TcTables&) = delete;
  TcTables& operator=(const TcTables&) = delete;
  ~TcTables() {
    cudaFree(sx0); cudaFree(hB); cudaFree(vB); cudaFree(vys); cudaFree(vcl); cudaFree(lut2);
  }
  bool ok = false;
  std::string why;  // why the request is outside the kernel's plan (then the mma.sync kernel runs)
  int KH = 0, KV = 0, NCH = 0, NCHmax = 0, nchunks = 0, nstrips = 0;
  int32_t* sx0 = nullptr;
  uint8_t* hB = nullptr;
  uint8_t* vB = nullptr;
  int32_t* vys = nullptr;
  int32_t* vcl = nullptr;
  uint32_t* lut2 = nullptr;
  std::vector<int32_t> hvys, hvcl;  // host copies (the kernel parameters carry them too)
};

struct TcKey {
  int dev, w, w2, h, h2, backend;
  uint32_t lut[768];
  bool operator<(const TcKey& o) const { return std::memcmp(this, &o, sizeof(TcKey)) < 0; }
};

std::mutex g_mu;
LruCache<TcKey, TcTables>* g_cache = new LruCache<TcKey, TcTables>(kTableCacheEntries);

// balanced base-256 digits: w = d2*2^16 + d1*2^8 + d0, d0 and d1 in [-128, 127]
void digits(int32_t w, int (&d)[3]) {
  d[0] = ((w & 255) ^ 128) - 128;
  const int32_t r = (w - d[0]) >> 8;
  d[1] = ((r & 255) ^ 128) - 128;
  d[2] = (r - d[1]) >> 8;
}

// K-major core-matrix offset of (n, k) in an [N][K] s8 operand (SWIZZLE_NONE)
inline size_t offk(int n, int k, int K) {
  return static_cast<size_t>(n / 8) * (K / 16) * 128 + static_cast<size_t>(k / 16) * 128 + (n % 8) * 16 + k % 16;
}

template <typename T>
cudaError_t upload(T** dst, const std::vector<T>& v) {
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(dst), std::max<size_t>(v.size(), 1) * sizeof(T));
  if (e != cudaSuccess) return e;
  return cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
}

fc_status build(const fc_plan_s* P, TcTables* t) {
  const AxisTable& th = *P->th;
  const AxisTable& tv = *P->tv;
  const int W2 = P->w2, H2 = P->h2, H = P->meta.height;
  const int nstrips = (W2 + kStrip - 1) / kStrip, gh2 = H2 / 28;
  t->nstrips = nstrips;
  t->nchunks = (H + kChunk - 1) / kChunk;
  // H: strip windows, KH (one more column than any tap reaches: the constant column)
  std::vector<int32_t> sx0(nstrips);
  int span = 0;
  for (int s = 0; s < nstrips; ++s) {
    const int X0 = s * kStrip, X1 = std::min(X0 + kStrip, W2);
    sx0[s] = th.xmin[X0] & ~15;
    for (int o = X0; o < X1; ++o) span = std::max(span, th.xmin[o] + th.cnt[o] - sx0[s]);
  }
  t->KH = (span + 1 + 31) & ~31;
  if (t->KH > 256) {
    t->why = "horizontal window wider than 255 source columns per strip";
    return FC_OK;
  }
  // V: half-band windows, KV, last chunk per band, ring depth
  std::vector<int32_t> vys(2 * gh2), vcl(gh2);
  int vspan = 0, bspan = 0;
  for (int hb = 0; hb < gh2; ++hb) {
    int bend = 0;
    for (int h = 0; h < 2; ++h) {
      const int r0 = 28 * hb + 16 * h, r1 = std::min(r0 + 16, 28 * hb + 28);
      const int ys = tv.xmin[r0] & ~7;
      int end = ys;
      for (int r = r0; r < r1; ++r) end = std::max(end, tv.xmin[r] + tv.cnt[r]);
      vys[2 * hb + h] = ys;
      vspan = std::max(vspan, end - ys);
      bend = std::max(bend, end);
    }
    vcl[hb] = std::min(t->nchunks - 1, (bend - 1) / kChunk);
    bspan = std::max(bspan, vcl[hb] - (vys[2 * hb] >> 4) + 1);
  }
  t->KV = (vspan + 31) & ~31;
  if (t->KV > 128) {
    t->why = "vertical window wider than 128 source rows per 16 output rows";
    return FC_OK;
  }
  t->NCH = std::max(3, bspan + 2);  // >= span + 1: the ring-free wait never waits on a band that needs the chunk being written
  // bands whose windows start within any NCH consecutive chunks: in flight between the
  // V MMAs and the H epilogue's ring-free wait (<= kNVD barrier slots, two runs' worth)
  int inflight = 0;
  for (int hb = 0; hb < gh2; ++hb) {
    int n = 0;
    for (int hb2 = hb; hb2 < gh2 && (vys[2 * hb2] >> 4) < (vys[2 * hb] >> 4) + t->NCH; ++hb2) ++n;
    inflight = std::max(inflight, n);
  }
  if (t->NCH + 2 > kNHR) {
    t->why = "ring deeper than the ready-barrier slots";
    return FC_OK;
  }
  if (2 * inflight + 2 > kNVD) {
    t->why = "too many bands per ring window";
    return FC_OK;
  }
  // the deepest ring the barrier slots allow (the launch uses what shared memory
  // leaves: a deeper ring lets the H epilogue run further ahead of the V pass)
  t->NCHmax = t->NCH;
  for (int nch = t->NCH + 1; nch + 2 <= kNHR; ++nch) {
    int n_in = 0;
    for (int hb = 0; hb < gh2; ++hb) {
      int n = 0;
      for (int hb2 = hb; hb2 < gh2 && (vys[2 * hb2] >> 4) < (vys[2 * hb] >> 4) + nch; ++hb2) ++n;
      n_in = std::max(n_in, n);
    }
    if (2 * n_in + 2 > kNVD) break;
    t->NCHmax = nch;
  }
  // every V output lands inside the doubled table: floor((S + 2^21) / 2^22) in [-48, 303]
  for (int o = 0; o < tv.out; ++o) {
    int64_t pos = 0, neg = 0;
    for (int k = 0; k < tv.cnt[o]; ++k) {
      const int64_t w = tv.iw[static_cast<size_t>(o) * tv.ksize + k];
      (w > 0 ? pos : neg) += w;
    }
    const int64_t vmax = ((1 << 21) + 255 * pos) >> 22, vmin = ((1 << 21) + 255 * neg) >> 22;
    if (vmin < -48 || vmax > 303) return fail(FC_ERR_UNSUPPORTED, "vertical resize weights reach outside the normalisation table");
  }
  // weight digits
  std::vector<uint8_t> hB(static_cast<size_t>(nstrips) * kNH * t->KH, 0);
  for (int s = 0; s < nstrips; ++s) {
    uint8_t* B = hB.data() + static_cast<size_t>(s) * kNH * t->KH;
    const int X0 = s * kStrip;
    for (int o = 0; o < kStripPad; ++o)
      for (int k = 0; k < t->KH; ++k) {
        const bool valid = o < kStrip && X0 + o < W2;
        int d[3] = {0, 0, 0};
        if (valid) digits(weight_at(th, X0 + o, sx0[s] + k), d);
        if (k == t->KH - 1) d[2] += 32;  // the constant column (A = 1): Pillow's 2^21
        for (int pl = 0; pl < 3; ++pl) {
          if (d[pl] < -128 || d[pl] > 127) return fail(FC_ERR_UNSUPPORTED, "weight digit out of s8 range");
          B[offk(pl * kStripPad + o, k, t->KH)] = static_cast<uint8_t>(static_cast<int8_t>(d[pl]));
        }
      }
  }
  const size_t bvh = static_cast<size_t>(kNV) * t->KV;  // bytes per half band
  std::vector<uint8_t> vB(static_cast<size_t>(gh2) * 2 * bvh, 0);
  for (int hb = 0; hb < gh2; ++hb)
    for (int h = 0; h < 2; ++h) {
      uint8_t* B = vB.data() + (static_cast<size_t>(hb) * 2 + h) * bvh;
      for (int jj = 0; jj < 16; ++jj) {
        const int yl = 16 * h + jj;
        for (int k = 0; k < t->KV; ++k) {
          int d[3] = {0, 0, 0};
          if (yl < 28) digits(weight_at(tv, 28 * hb + yl, vys[2 * hb + h] + k), d);
          for (int pl = 0; pl < 3; ++pl) {
            if (d[pl] < -128 || d[pl] > 127) return fail(FC_ERR_UNSUPPORTED, "weight digit out of s8 range");
            B[offk(pl * 16 + jj, k, t->KV)] = static_cast<uint8_t>(static_cast<int8_t>(d[pl]));
          }
        }
      }
    }
  std::vector<uint32_t> lut2(3 * kLut2N);
  for (int c = 0; c < 3; ++c)
    for (int i = 0; i < kLut2N; ++i) {
      const int v = std::min(255, std::max(0, (i - (kLut2Lo - 1)) >> 1));  // floor((a + 1) / 2), a = i - 97
      lut2[c * kLut2N + i] = P->lut_dev[c * 256 + v];
    }
  t->hvys = vys;
  t->hvcl = vcl;
  cudaError_t e = upload(&t->sx0, sx0);
  if (e == cudaSuccess) e = upload(&t->hB, hB);
  if (e == cudaSuccess) e = upload(&t->vB, vB);
  if (e == cudaSuccess) e = upload(&t->vys, vys);
  if (e == cudaSuccess) e = upload(&t->vcl, vcl);
  if (e == cudaSuccess) e = upload(&t->lut2, lut2);
  if (e != cudaSuccess) {  // the caller's shared_ptr frees what was uploaded
    return e == cudaErrorMemoryAllocation ? fail(FC_ERR_OOM, "tcgen05 table upload: out of device memory")
                                          : cuda_fail(e, "tcgen05 table upload");
  }
  t->ok = true;
  return FC_OK;
}

fc_status tables(fc_plan_s* P, int dev, const TcTables** out) {
  {
    std::lock_guard<std::mutex> lk(P->mu);
    auto it = P->tc.find(dev);
    if (it != P->tc.end()) {
      *out = static_cast<const TcTables*>(it->second.get());
      return FC_OK;
    }
  }
  TcKey key;
  std::memset(&key, 0, sizeof(key));
  key.dev = dev;
  key.w = P->th->in;
  key.w2 = P->th->out;
  key.h = P->tv->in;
  key.h2 = P->tv->out;
  key.backend = P->cfg.backend;
  std::memcpy(key.lut, P->lut_dev.data(), sizeof(key.lut));
  std::lock_guard<std::mutex> gk(g_mu);
  std::shared_ptr<TcTables> sp = g_cache->get(key);
  if (!sp) {
    sp = std::make_shared<TcTables>();
    const fc_status st = build(P, sp.get());
    if (st != FC_OK) return st;
    g_cache->put(key, sp);
  }
  std::lock_guard<std::mutex> lk(P->mu);
  *out = sp.get();
  P->tc[dev] = std::move(sp);
  return FC_OK;
}

inline int up1024(int x) { return (x + 1023) & ~1023; }

}  // namespace
}  // namespace tc

fc_status launch_tc(fc_plan_s* P, const std::vector<Job>& jobs, void* stream, uint8_t* dbg_src, uint8_t* dbg_rs,
                    bool* handled, bool dry) {
  using namespace tc;
  *handled = false;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return FC_OK;
  int major = 0, max_smem = 0, nsm = 0;
  device_attrs(dev, &major, &max_smem, &nsm);
  if (major != 10) return FC_OK;  // the caller reports the missing sm_100 device
  const TcTables* t = nullptr;
  fc_status st = tables(P, dev, &t);
  if (st != FC_OK) {
    *handled = true;
    return st;
  }
  if (!t->ok || nsm < t->nstrips || P->h2 / 28 > kMaxBands) return FC_OK;
  const bool verbose = std::getenv("FC_VERBOSE") != nullptr;

  static thread_local TcParams prm;  // ~31 KB: keep it off the stack
  std::memset(&prm, 0, offsetof(TcParams, tm));
  prm.W = P->meta.width;
  prm.H = P->meta.height;
  prm.W2 = P->w2;
  prm.H2 = P->h2;
  prm.gh2 = static_cast<int>(P->gh / 2);
  prm.gw2 = static_cast<int>(P->gw / 2);
  prm.nstrips = t->nstrips;
  prm.KH = t->KH;
  prm.KV = t->KV;
  prm.BW = t->KH;
  prm.nchunks = t->nchunks;
  prm.rawb = 48 * prm.BW;
  prm.sbo_a = (prm.KH / 16) * kLboA;
  prm.ahb = 16 * prm.sbo_a;
  prm.bvb = 2 * kNV * prm.KV;
  // shared-memory plan: deepest A_H / raw / B_V pipelines that fit, then the
  // deepest ring that still fits
  int smem = 0;
  auto plan = [&](int na, int nr, int nbv, int nch, bool commit) -> int {
    int off = 1024;  // barriers + TMEM slot
    const int off_lut = off;
    off = up1024(off + 3 * kLut2N * 4);
    const int off_raw = off;
    off = up1024(off + nr * prm.rawb);
    const int off_ah = off;
    off = up1024(off + na * prm.ahb);
    const int off_bh = off;
    off = up1024(off + kNH * prm.KH);
    const int off_bv = off;
    off = up1024(off + nbv * prm.bvb);
    const int off_ring = off;
    off += 24 * (nch + 2) * 256;
    const int off_tab = off;
    off += (3 * prm.gh2 * 4 + 15) & ~15;
    const int total = off + 1024;  // the kernel aligns its base up to 1024
    if (commit) {
      prm.NR = nr;
      prm.NA = na;
      prm.NBV = nbv;
      prm.NCH = nch;
      prm.sbo_v = (nch + 2) * 256;
      prm.off_lut = off_lut;
      prm.off_raw = off_raw;
      prm.off_ah = off_ah;
      prm.off_bh = off_bh;
      prm.off_bv = off_bv;
      prm.off_ring = off_ring;
      prm.off_tab = off_tab;
    }
    return total;
  };
  for (int na = 3; na >= 1 && !smem; --na)
    for (int nr = 4; nr >= 2 && !smem; --nr)
      for (int nbv = kMaxBV; nbv >= 2 && !smem; --nbv)
        if (plan(na, nr, nbv, t->NCH, false) <= max_smem) {
          int nch = t->NCH;
          while (nch < t->NCHmax && plan(na, nr, nbv, nch + 1, false) <= max_smem) ++nch;
          smem = plan(na, nr, nbv, nch, true);
        }
  if (!smem) return FC_OK;
  *handled = true;
  for (int i = 0; i < 2 * prm.gh2; ++i) prm.cvys[i] = static_cast<uint16_t>(t->hvys[i]);
  for (int i = 0; i < prm.gh2; ++i) prm.cvcl[i] = static_cast<uint16_t>(t->hvcl[i]);
  prm.sx0 = t->sx0;
  prm.hB = t->hB;
  prm.vB = t->vB;
  prm.vys = t->vys;
  prm.vcl = t->vcl;
  prm.lut2 = t->lut2;
  color_words(P->cfg.color, &prm.ckR, &prm.ckG, &prm.ckGv, &prm.ckB, &prm.cbR, &prm.cbG, &prm.cbB);
  prm.dbg_src = dbg_src;
  prm.dbg_rs = dbg_rs;
  const int64_t nfj = static_cast<int64_t>(jobs[0].frames.size());
  const int64_t nf = nfj * static_cast<int64_t>(jobs.size());
  const long long items = (nf / 2) * static_cast<long long>(prm.gh2);
  if (items > INT32_MAX) return fail(FC_ERR_UNSUPPORTED, "launch too large (> 2^31 work items)");
  prm.nframes = static_cast<int>(nf);
  prm.npairs = static_cast<int>(nf / 2);
  prm.ppj = static_cast<int>(nfj / 2);
  prm.tokens = jobs[0].tokens;
  const bool inline_maps = jobs.size() == 1 && nf <= kMaxInline;
  std::vector<CUtensorMap> maps(inline_maps ? 0 : 2 * nf);
  CUtensorMap* mp = inline_maps ? prm.tm : maps.data();
  for (size_t j = 0; j < jobs.size(); ++j)
    for (int64_t i = 0; i < nfj; ++i) {
      const fc_nv12_surface& sf = jobs[j].surfaces[jobs[j].frames[i]];
      const int64_t fi = static_cast<int64_t>(j) * nfj + i;
      st = tensor_map(sf.y, sf.pitch_y, prm.H, prm.BW, kChunk, &mp[2 * fi]);
      if (st == FC_OK) st = tensor_map(sf.uv, sf.pitch_uv, prm.H / 2, prm.BW, kChunk / 2, &mp[2 * fi + 1]);
      if (st != FC_OK) return st;
    }
  if (dry) return FC_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  void* desc = nullptr;
  if (!inline_maps) {  // descriptor sections: [tensor maps | per-job token bases]
    const size_t mbytes = maps.size() * sizeof(CUtensorMap);
    const size_t tbytes = jobs.size() > 1 ? jobs.size() * sizeof(void*) : 0;
    std::vector<uint8_t> host(mbytes + tbytes);
    std::memcpy(host.data(), maps.data(), mbytes);
    for (size_t j = 0; j < jobs.size() && tbytes; ++j)
      std::memcpy(host.data() + mbytes + j * sizeof(void*), &jobs[j].tokens, sizeof(void*));
    cudaMemPool_t pool = descriptor_pool(dev);
    e = pool ? cudaMallocFromPoolAsync(&desc, host.size(), pool, s) : cudaMallocAsync(&desc, host.size(), s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync (launch descriptor)");
    e = cudaMemcpyAsync(desc, host.data(), host.size(), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) {
      cudaFreeAsync(desc, s);
      return cuda_fail(e, "descriptor upload");
    }
    prm.tmg = reinterpret_cast<const CUtensorMap*>(desc);
    if (tbytes) prm.tokj = reinterpret_cast<void* const*>(static_cast<uint8_t*>(desc) + mbytes);
  }
  TcKernelFn fprod = nullptr, fdbg = nullptr, fprof = nullptr;
  tc_kernels(&fprod, &fdbg, &fprof);
  // FC_TC_PROF=1 (experiments): the instance that counts each warp's barrier-wait cycles
  const bool profile = std::getenv("FC_TC_PROF") != nullptr && !(dbg_src || dbg_rs);
  TcKernelFn fn = (dbg_src || dbg_rs) ? fdbg : profile ? fprof : fprod;
  st = ensure_smem_attr(dev, reinterpret_cast<const void*>(fn), static_cast<size_t>(smem));
  if (st != FC_OK) {
    if (desc) cudaFreeAsync(desc, s);
    return st;
  }
  // one CTA per SM (512 TMEM columns each); every strip needs at least one CTA
  const long long work = static_cast<long long>(prm.npairs) * prm.gh2 * t->nstrips;
  const int grid = static_cast<int>(std::max<long long>(t->nstrips, std::min<long long>(nsm, work)));
  if (verbose)
    std::fprintf(stderr, "fc tc: KH %d KV %d NCH %d NR %d NA %d NBV %d smem %d grid %d strips %d pairs %d\n", prm.KH,
                 prm.KV, prm.NCH, prm.NR, prm.NA, prm.NBV, smem, grid, t->nstrips, prm.npairs);
  if (profile && std::getenv("FC_TC_ABLATE")) prm.ablate = std::atoi(std::getenv("FC_TC_ABLATE"));
  unsigned long long* prof = nullptr;
  if (profile && cudaMalloc(&prof, sizeof(unsigned long long) * 9 * kWarps * grid) == cudaSuccess) {
    cudaMemsetAsync(prof, 0, sizeof(unsigned long long) * 9 * kWarps * grid, s);
    prm.prof = prof;
  }
  fn<<<grid, kThreads, smem, s>>>(prm);
  e = cudaGetLastError();
  if (prof) {  // per role: mean fraction of the warp's lifetime spent in each wait site
    std::fprintf(stderr, "fc tc prof: ablate %d (env %s)\n", prm.ablate,
                 std::getenv("FC_TC_ABLATE") ? std::getenv("FC_TC_ABLATE") : "-");
    prm.prof = nullptr;
    prm.ablate = 0;
    std::vector<unsigned long long> h(9 * kWarps * grid);
    cudaMemcpyAsync(h.data(), prof, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    cudaFree(prof);
    struct Role { const char* name; int w0, w1; const char* sites; };
    const Role roles[] = {{"V-epi", kVEpi0, kVEpi0 + 8, "vfull"}, {"H-epi", kHEpiWarpA, kHEpiWarpA + 3, "vdone hfull"},
                          {"H-epi'", kHEpiWarpB, kHEpiWarpB + 3, "vdone hfull"},
                          {"H-MMA", kMmaWarp, kMmaWarp + 1, "bh hempty afull | [5] H issue"},
                          {"V-MMA", kVMmaWarp, kVMmaWarp + 1, "- hready bvfull vempty | [6] V issue"},
                          {"TMA", kTmaWarp, kTmaWarp + 1, "bvempty rawempty"},
                          {"colour", kColWarp0, kColWarp0 + kColWarps, "rawfull aempty"}};
    for (const Role& r : roles) {
      double acc[9] = {0};
      int n = 0;
      for (int b = 0; b < grid; ++b)
        for (int w = r.w0; w < r.w1; ++w, ++n)
          for (int k = 0; k < 9; ++k) acc[k] += static_cast<double>(h[(static_cast<size_t>(b) * kWarps + w) * 9 + k]);
      std::fprintf(stderr, "fc tc prof %-7s (%s): total %.0f cyc/warp, waits", r.name, r.sites, acc[8] / n);
      for (int k = 0; k < 8; ++k)
        if (acc[k] > 0) std::fprintf(stderr, " [%d] %.3f", k, acc[k] / acc[8]);
      std::fprintf(stderr, "\n");
    }
  }
  if (desc) cudaFreeAsync(desc, s);
  if (e != cudaSuccess) return cuda_fail(e, "tcgen05 kernel launch");
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  last_kernel() = FC_KERNEL_TC;
  return FC_OK;
}

}  // namespace fc
