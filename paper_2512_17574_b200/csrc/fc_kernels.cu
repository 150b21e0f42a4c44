// fc_kernels.cu -- host side of the fused kernel: device tables (MMA
// fragments, windows, LUT), strip geometry, TMA tensor maps, launch
// descriptors and the fc_preprocess / fc_preprocess_debug /
// fc_preprocess_batch entry points.  The kernel itself is fc_fused.cuh.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "fc_fused.cuh"
#include "fc_internal.h"
#include "fc_launch.h"

namespace fc {

// ------------------------------------------------------------------ host side

// Instances: k-steps (32 source pixels each) of the H-pass and V-pass MMA
// windows, KSH, KSV in 1..4.  8 consecutive outputs need KS*32 >= span + 3
// (4-byte alignment).
static const Instance* instances() {
  static Instance tab[16];
  static bool init = [] {
    instances_ksh1(tab);
    instances_ksh2(tab + 4);
    instances_ksh3(tab + 8);
    instances_ksh4(tab + 12);
    return true;
  }();
  (void)init;
  return tab;
}
constexpr int kMaxKS = 4;

fc_status cuda_fail(cudaError_t e, const char* what) {
  return fail(FC_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename T>
static cudaError_t upload(T** dst, const std::vector<T>& v) {
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(dst), std::max<size_t>(v.size(), 1) * sizeof(T));
  if (e != cudaSuccess) return e;
  return cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
}

// Integer Pillow weight of output o at source index src (0 outside the window).
int32_t weight_at(const AxisTable& t, int o, int src) {
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
// (g = lane/4, t = lane%4) holds MMA k = ks*32 + 16 r + 4 t + [0..3] of output
// g.  V: MMA k is source index xs + k.  H (kperm): the kernel loads A with one
// LDS.64 per row, so MMA k = ks*32 + 16 r + 4 t + b is source index
// xs + ks*32 + 8 t + 4 r + b.
static void frag_group(const AxisTable& t, const int (&outs)[8], int xs, int KS, uint32_t* dst, bool kperm) {
  for (int ks = 0; ks < KS; ++ks)
    for (int pl = 0; pl < 3; ++pl)
      for (int lane = 0; lane < 32; ++lane)
        for (int rr = 0; rr < 2; ++rr) {
          const int g = lane >> 2, tq = lane & 3;
          uint32_t word = 0;
          for (int bb = 0; bb < 4; ++bb) {
            const int k = ks * 32 + (kperm ? 8 * tq + 4 * rr : 16 * rr + 4 * tq) + bb;
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
  // V groups: MMA N column n is output row pi(n) of the 8-row group, pi(2t) = t,
  // pi(2t+1) = t + 4 (the kernel's j0 / j1: compact 4-row LUT footprints)
  auto v_outs = [&](int grp, int (&outs)[8]) {
    const int hb = grp / 4, gi = grp % 4;
    for (int n = 0; n < 8; ++n) {
      const int row = 8 * gi + (n >> 1) + 4 * (n & 1);
      outs[n] = row < 28 ? 28 * hb + row : -1;
    }
  };
  int ksh = 1, ksv = 1;
  for (int tt = 0; tt < nth; ++tt) {
    int outs[8];
    h_outs(tt, outs);
    const int first = std::min(tt / htiles * sw + 8 * (tt % htiles), th.out - 1);
    m->hxs[tt] = th.xmin[first] & ~7;  // 8 columns = 16 bytes of a row-pair line: aligned LDS.128 A loads
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
    frag_group(th, outs, m->hxs[tt], ksh, &m->hfr[static_cast<size_t>(tt) * ksh * 3 * 64], true);
  }
  for (int grp = 0; grp < gh2 * 4; ++grp) {
    int outs[8];
    v_outs(grp, outs);
    frag_group(tv, outs, m->vys[grp], ksv, &m->vfr[static_cast<size_t>(grp) * ksv * 3 * 64], false);
  }
}

// Process-wide cache of uploaded tables, keyed by everything the tables are a
// function of (device, W->W', H->H', normalisation).  Plans of equally shaped
// requests share one upload, so fc_plan + fc_preprocess never touch the device
// synchronously after the first request of a shape.
struct TableKey {
  int dev, sw, w, w2, h, h2, backend;
  uint32_t lut_bits[768];
  bool operator<(const TableKey& o) const { return std::memcmp(this, &o, sizeof(TableKey)) < 0; }
};

static std::mutex g_tables_mu;
static LruCache<TableKey, DeviceTables>* g_tables = new LruCache<TableKey, DeviceTables>(kTableCacheEntries);

DeviceTables::~DeviceTables() {
  cudaFree(hx); cudaFree(hxs); cudaFree(hfr); cudaFree(vx); cudaFree(vcnt); cudaFree(vys); cudaFree(vfr); cudaFree(lut);
}

static fc_status device_tables(fc_plan_s* P, int dev, int sw, const DeviceTables** out) {
  std::lock_guard<std::mutex> lk(P->mu);
  const int pkey = dev * 1024 + sw;
  auto it = P->dev.find(pkey);
  if (it != P->dev.end()) {
    *out = it->second.get();
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
  key.backend = P->cfg.backend;
  std::memcpy(key.lut_bits, P->lut_dev.data(), sizeof(key.lut_bits));
  std::lock_guard<std::mutex> gk(g_tables_mu);
  if (std::shared_ptr<DeviceTables> hit = g_tables->get(key)) {
    *out = hit.get();
    P->dev[pkey] = std::move(hit);
    return FC_OK;
  }
  // every V output must land inside the extended table: floor(S / 2^22) with
  // S = 2^21 + sum T*iv over u8 T lies in [vmin, vmax] below.  For Pillow's
  // bicubic (a = -0.5) the negative lobes of the normalised filter sum to about
  // 1/8 at most (2x upscale phase): v in [-34, 289] over tests/test_plan.py's
  // sweep; checked here per plan, not assumed
  {
    const AxisTable& tv = *P->tv;
    for (int o = 0; o < tv.out; ++o) {
      int64_t pos = 0, neg = 0;
      for (int k = 0; k < tv.cnt[o]; ++k) {
        const int64_t w = tv.iw[static_cast<size_t>(o) * tv.ksize + k];
        (w > 0 ? pos : neg) += w;
      }
      const int64_t vmax = ((1 << 21) + 255 * pos) >> 22, vmin = ((1 << 21) + 255 * neg) >> 22;
      if (vmin < -kLutLo || vmax >= 256 + kLutLo)
        return fail(FC_ERR_UNSUPPORTED, "vertical resize weights reach outside the normalisation table");
    }
  }
  MmaTables m;
  build_mma_tables(P, sw, &m);
  if (m.ksh > kMaxKS || m.ksv > kMaxKS)
    return fail(FC_ERR_UNSUPPORTED, "resize window wider than 128 source pixels per 8 outputs");
  auto sp = std::make_shared<DeviceTables>();  // frees whatever was uploaded if this fails
  DeviceTables& t = *sp;
  static std::atomic<uint64_t> serials{0};
  t.serial = ++serials;
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
  // extended normalisation table (kernel: kLutLo entries below v = 0 and above
  // v = 255 repeat the end values, so the V pass needs no clamp)
  std::vector<uint32_t> lut_ext(3 * kLutN);
  for (int c = 0; c < 3; ++c)
    for (int i = 0; i < kLutN; ++i)
      lut_ext[c * kLutN + i] = P->lut_dev[c * 256 + std::min(255, std::max(0, i - kLutLo))];
  if (e == cudaSuccess) e = upload(&t.lut, lut_ext);
  if (e != cudaSuccess)
    return e == cudaErrorMemoryAllocation ? fail(FC_ERR_OOM, "table upload: out of device memory")
                                          : cuda_fail(e, "table upload");
  g_tables->put(key, sp);
  *out = sp.get();
  P->dev[pkey] = std::move(sp);
  return FC_OK;
}

struct Geometry {
  int sw, htiles, SWPN, SWP, BW, NX, TR, TRW, nstrips, nchunks;
  KernelFn fn, fn_dbg, fn_bf16, fn_u8, fn_paged, fn_paged_bf16, fn_i420, fn_i420_dbg, fn_cols;
  size_t smem;   // at nstages
  int nstages;   // raw TMA stages: 4, or 2 when that buys another CTA per SM (wide-window configs)
};

static size_t smem_bytes(int stages, int SWP, int RAWW, int TRW) {
  return kLutBytes + 128 + static_cast<size_t>(stages) * 48 * RAWW + static_cast<size_t>(6) * kChunkRows * SWP +
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
    const int SX0 = th.xmin[X0] & (P->cfg.surface_format == FC_SURFACE_I420 ? ~31 : ~15);  // == the kernel's sxmask
    for (int i = 0; i < g->htiles && X0 + 8 * i < X1; ++i)
      need = std::max(need, (th.xmin[X0 + 8 * i] & ~7) - SX0 + 32 * dt->ksh);
    for (int o = X0; o < X1; ++o) taps = std::max(taps, th.xmin[o] + th.cnt[o] - SX0);
  }
  // converted width; I420 loads U and V boxes of SWPN/2 bytes, which TMA wants
  // in multiples of 16
  const int cq = P->cfg.surface_format == FC_SURFACE_I420 ? 32 : 16;
  need = std::max(need, (taps + cq - 1) / cq * cq);  // the converted width (SWPN) fits every row
  // round up to 8 mod 16: the H pass's LDS.64 A loads of a half-warp read rows
  // 0, 4, 8, 12 (or 2, 6, 10, 14) of a chunk, 32 B each; with a row stride of
  // 8 mod 16 bytes those land in distinct quarters of the 128-B bank space
  const int swp8 = (need + 7) / 8 * 8;
  const int swpb = swp8 % 16 == 8 ? swp8 : swp8 + 8;
  g->SWPN = ((taps + cq - 1) / cq) * cq;
  g->SWP = swpb;
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
  for (int ii = 0; ii < 16; ++ii) {
    const Instance& in = instances()[ii];
    if (in.ksh == dt->ksh && in.ksv == dt->ksv) {
      g->fn = in.fn;
      g->fn_dbg = in.fn_dbg;
      g->fn_bf16 = in.fn_bf16;
      g->fn_u8 = in.fn_u8;
      g->fn_paged = in.fn_paged;
      g->fn_paged_bf16 = in.fn_paged_bf16;
      g->fn_i420 = in.fn_i420;
      g->fn_i420_dbg = in.fn_i420_dbg;
      g->fn_cols = in.fn_cols;
    }
  }
  if (!g->fn) return fail(FC_ERR_UNSUPPORTED, "no kernel instance for this resize window");
  if (dt->ksh <= 2 && 2 * kChunkRows * (g->SWPN / 16) > 2 * kComputeThreads)
    return fail(FC_ERR_UNSUPPORTED, "colour stage: more than 2 items per thread");
  g->nstages = kMaxStages;
  g->smem = smem_bytes(kMaxStages, g->SWP, g->BW * g->NX, g->TRW);
  if (g->smem > static_cast<size_t>(max_smem)) {
    g->nstages = 2;
    g->smem = smem_bytes(2, g->SWP, g->BW * g->NX, g->TRW);
  }
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
fc_status tensor_map(const uint8_t* base, int64_t pitch, int64_t rows, int bw, int bh, CUtensorMap* out) {
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
void color_words(fc_color m, uint32_t* kR, uint32_t* kG, uint32_t* kGv, uint32_t* kB, int* bR, int* bG, int* bB) {
  struct K { int y, y0, rv, gu, gv, bu; };
  static const K kTab[4] = {
      {298, 16, 409, -100, -208, 516},  // BT.601 limited (R3)
      {298, 16, 459, -55, -136, 541},   // BT.709 limited
      {256, 0, 359, -88, -183, 454},    // BT.601 full
      {256, 0, 403, -48, -120, 475},    // BT.709 full
  };
  const K& k = kTab[static_cast<int>(m)];
  auto pack = [](int hi, int lo) { return (static_cast<uint32_t>(hi & 0xFFFF) << 16) | static_cast<uint32_t>(lo & 0xFFFF); };
  *kR = pack(k.rv, k.y);
  *kB = pack(k.bu, k.y);
  *kG = pack(k.gu, k.y);
  *kGv = pack(k.gv, 0);
  *bR = -k.y0 * k.y - 128 * k.rv + 128;
  *bG = -k.y0 * k.y - 128 * (k.gu + k.gv) + 128;
  *bB = -k.y0 * k.y - 128 * k.bu + 128;
}
static void color_constants(fc_color m, Params* p) {
  color_words(m, &p->ckR, &p->ckG, &p->ckGv, &p->ckB, &p->cbR, &p->cbG, &p->cbB);
}

// The rank's frame list (its sampled frames, then pad copies of the last),
// after validating every surface it reads.  Empty for a rank with no rows.
int32_t& last_kernel() {  // fc_last_kernel(): the calling thread's last fused-kernel launch
  static thread_local int32_t k = FC_KERNEL_NONE;
  return k;
}

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
  const bool i420 = P->cfg.surface_format == FC_SURFACE_I420;
  const int cw = i420 ? W / 2 : W;  // chroma plane bytes per row
  for (int64_t f : *frames) {
    if (f >= num_surfaces) return fail(FC_ERR_MISSING_SURFACE, "surface array too short for frame " + std::to_string(f));
    const fc_nv12_surface& s = surfaces[f];
    if (!s.y || !s.uv || (i420 && !s.v)) return fail(FC_ERR_MISSING_SURFACE, "NULL surface for frame " + std::to_string(f));
    if ((reinterpret_cast<uintptr_t>(s.y) & 15) || (reinterpret_cast<uintptr_t>(s.uv) & 15) ||
        (i420 && (reinterpret_cast<uintptr_t>(s.v) & 15)))
      return fail(FC_ERR_UNSUPPORTED, "surface planes must be 16-byte aligned");
    if ((s.pitch_y & 15) || (s.pitch_uv & 15) || s.pitch_y < W || s.pitch_uv < cw || s.pitch_y > INT32_MAX ||
        s.pitch_uv > INT32_MAX)
      return fail(FC_ERR_UNSUPPORTED, "pitches must be multiples of 16, pitch_y >= width, pitch_uv >= chroma width");
  }
  return FC_OK;
}


// ONE persistent launch over every pair of `jobs` (all of P's geometry and
// pair count).  Up to kMaxInlineFrames frames of a single job, the tensor maps
// travel in the kernel parameters (nothing to upload; graph-capturable);
// beyond that, or for several jobs, a descriptor [maps | per-job token bases]
// is copied to a stream-ordered device allocation (cudaMallocAsync, freed
// after the launch in stream order).
// Library-owned stream-ordered pool for launch descriptors: the release
// threshold keeps freed blocks in the pool across synchronisations, so a
// steady stream of requests never goes back to the driver for memory (the
// default pool returns memory at every sync).
cudaMemPool_t descriptor_pool(int dev) {
  static std::mutex mu;
  static std::map<int, cudaMemPool_t>* pools = new std::map<int, cudaMemPool_t>();
  std::lock_guard<std::mutex> lk(mu);
  auto it = pools->find(dev);
  if (it != pools->end()) return it->second;
  cudaMemPoolProps props{};
  props.allocType = cudaMemAllocationTypePinned;
  props.handleTypes = cudaMemHandleTypeNone;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  cudaMemPool_t pool = nullptr;
  if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) return nullptr;
  uint64_t keep = UINT64_MAX;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  (*pools)[dev] = pool;
  return pool;
}

// Launch configurations (geometry, TMA stages, occupancy) per (table set,
// kernel instance, surface format): requests of a known shape skip the
// geometry search and the occupancy queries (host cost of a small request).
struct LaunchKey {
  uint64_t serial;
  const void* fn;
  int i420;
  bool operator==(const LaunchKey& o) const { return serial == o.serial && fn == o.fn && i420 == o.i420; }
};
struct LaunchKeyHash {
  size_t operator()(const LaunchKey& k) const {
    return std::hash<uint64_t>()(k.serial) ^ (std::hash<const void*>()(k.fn) << 1) ^ static_cast<size_t>(k.i420);
  }
};
struct LaunchCfg {
  Geometry g;
  int occ;
};
static std::mutex g_launch_mu;
static std::unordered_map<LaunchKey, LaunchCfg, LaunchKeyHash>* g_launch =
    new std::unordered_map<LaunchKey, LaunchCfg, LaunchKeyHash>();

}  // namespace fc
namespace fc {
// Device attributes the launch path needs, queried once per device.
void device_attrs(int dev, int* major, int* max_smem, int* nsm) {
  static std::mutex mu;
  static std::map<int, std::array<int, 3>>* cache = new std::map<int, std::array<int, 3>>();
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache->find(dev);
  if (it == cache->end()) {
    std::array<int, 3> a{0, 0, 0};
    cudaDeviceGetAttribute(&a[0], cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&a[1], cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&a[2], cudaDevAttrMultiProcessorCount, dev);
    it = cache->emplace(dev, a).first;
  }
  *major = it->second[0];
  *max_smem = it->second[1];
  *nsm = it->second[2];
}

// cudaFuncAttributeMaxDynamicSharedMemorySize only ever grows per (device,
// kernel), so a launch never sees a smaller limit set for another shape.
fc_status ensure_smem_attr(int dev, const void* fn, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t>* cur = new std::map<std::pair<int, const void*>, size_t>();
  std::lock_guard<std::mutex> lk(mu);
  size_t& have = (*cur)[{dev, fn}];
  if (have >= smem) return FC_OK;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
  have = smem;
  return FC_OK;
}

// dry: validate and prepare everything (tables, geometry, tensor maps) but
// enqueue nothing -- fc_preprocess_batch checks every group before the first launch
static fc_status launch_jobs(fc_plan_s* P, const std::vector<Job>& jobs, void* stream, uint8_t* dbg_src,
                             uint8_t* dbg_rs, const fc_paged_tokens* paged = nullptr, bool colsplit = false,
                             bool dry = false) {
  // FC_TC=1 routes NV12 / fp32 requests whose windows fit its shared-memory
  // plan to the tcgen05 kernel (fc_tc.cu); by default this kernel runs them:
  // it is faster on every BASELINE config
  if (!paged && !colsplit && P->cfg.token_dtype == FC_TOKENS_F32 && P->cfg.surface_format == FC_SURFACE_NV12) {
    const char* env = std::getenv("FC_TC");
    if (env && std::atoi(env) != 0) {
      bool handled = false;
      const fc_status st = launch_tc(P, jobs, stream, dbg_src, dbg_rs, &handled, dry);
      if (handled) return st;
    }
  }
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  int major = 0, max_smem = 0, nsm = 0;
  device_attrs(dev, &major, &max_smem, &nsm);
  if (major != 10) return fail(FC_ERR_CUDA, "fc kernels are built for sm_100a only (no CPU/other-arch fallback)");
  const int W = P->meta.width, H = P->meta.height;
  // strips of 2 merge blocks; 1 merge block when a very wide resize window
  // would not fit the working set in shared memory
  const DeviceTables* dt = nullptr;
  Geometry g;
  fc_status st = FC_OK;
  const int i420k = P->cfg.surface_format == FC_SURFACE_I420 ? 1 : 0;
  for (int sw : {kStrip, 28}) {
    st = device_tables(P, dev, sw, &dt);
    if (st != FC_OK) return st;
    // geometry per (table set, surface format), searched once (a failed
    // search is remembered too: the caller then tries narrower strips)
    const LaunchKey gkey{dt->serial, nullptr, i420k};
    {
      std::lock_guard<std::mutex> lk(g_launch_mu);
      auto it = g_launch->find(gkey);
      if (it != g_launch->end()) {
        g = it->second.g;
        st = it->second.occ ? FC_OK : FC_ERR_UNSUPPORTED;
        if (st == FC_OK) break;
        continue;
      }
    }
    st = choose_geometry(P, dt, sw, max_smem, &g);
    {
      std::lock_guard<std::mutex> lk(g_launch_mu);
      (*g_launch)[gkey] = LaunchCfg{g, st == FC_OK ? 1 : 0};
    }
    if (st == FC_OK) break;
  }
  if (st != FC_OK) return st;
  const fc_token_dtype td = P->cfg.token_dtype;
  if (td != FC_TOKENS_F32 && (dbg_src || dbg_rs))
    return fail(FC_ERR_UNSUPPORTED, "debug dumps are built for fp32 tokens only");
  if (paged && (td == FC_TOKENS_U8 || jobs.size() != 1))
    return fail(FC_ERR_UNSUPPORTED, "paged output: one job, F32 or BF16 tokens");
  const bool i420 = P->cfg.surface_format == FC_SURFACE_I420;
  if (i420 && (td != FC_TOKENS_F32 || paged || colsplit))
    return fail(FC_ERR_UNSUPPORTED, "I420 surfaces: fp32 tokens, linear output (other variants are built for NV12)");
  if (colsplit && (td != FC_TOKENS_F32 || paged || dbg_src || dbg_rs || jobs.size() != 1))
    return fail(FC_ERR_UNSUPPORTED, "column-split output: one job, fp32 tokens, NV12");
  KernelFn fn = colsplit                 ? g.fn_cols
                : i420                   ? ((dbg_src || dbg_rs) ? g.fn_i420_dbg : g.fn_i420)
                : (dbg_src || dbg_rs)    ? g.fn_dbg
                : paged                ? (td == FC_TOKENS_BF16 ? g.fn_paged_bf16 : g.fn_paged)
                : td == FC_TOKENS_BF16 ? g.fn_bf16
                : td == FC_TOKENS_U8   ? g.fn_u8
                                       : g.fn;
  int occ = 0;
  const LaunchKey lkey{dt->serial, reinterpret_cast<const void*>(fn), i420 ? 1 : 0};
  bool cached = false;
  {
    std::lock_guard<std::mutex> lk(g_launch_mu);
    auto it = g_launch->find(lkey);
    if (it != g_launch->end()) {
      g = it->second.g;
      occ = it->second.occ;
      cached = true;
    }
  }
  if (!cached) {
    st = ensure_smem_attr(dev, reinterpret_cast<const void*>(fn), g.smem);
    if (st != FC_OK) return st;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kThreads, g.smem);
    if (e != cudaSuccess || occ < 1) return cuda_fail(e, "occupancy query");
    if (g.nstages == kMaxStages) {
      // a shallower TMA pipeline (2 stages) when it buys another CTA per SM:
      // latency hiding across CTAs is worth more than 2 extra chunks in flight
      const size_t smem2 = smem_bytes(2, g.SWP, g.BW * g.NX, g.TRW);
      int occ2 = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, fn, kThreads, smem2) == cudaSuccess && occ2 > occ) {
        g.nstages = 2;
        g.smem = smem2;
        occ = occ2;
      }
    }
    std::lock_guard<std::mutex> lk(g_launch_mu);
    if (g_launch->size() > 4096) g_launch->clear();
    (*g_launch)[lkey] = LaunchCfg{g, occ};
  }

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
  prm.nstages = g.nstages;
  prm.stage_shift = g.nstages == 4 ? 2 : 1;
  const int64_t nfj = static_cast<int64_t>(jobs[0].frames.size());
  const int64_t nf = nfj * static_cast<int64_t>(jobs.size());
  const long long items = (nf / 2) * static_cast<long long>(g.nstrips) * prm.gh2;
  if (items > INT32_MAX) return fail(FC_ERR_UNSUPPORTED, "launch too large (> 2^31 work items)");
  prm.frame_base = 0;
  prm.nframes = static_cast<int>(nf);
  prm.npairs = static_cast<int>(nf / 2);
  prm.ppj = static_cast<int>(nfj / 2);
  prm.tokens = paged ? paged->pool : jobs[0].tokens;
  if (colsplit) {  // [W][rows][C] column blocks of this launch's rows
    prm.cs_C = kCols / P->world;
    prm.cs_bstride = static_cast<long long>(nf / 2) * prm.gh2 * prm.gw2 * 4 * prm.cs_C;
    prm.cs_magic = static_cast<uint32_t>(((1ull << 32) + prm.cs_C - 1) / prm.cs_C);
  }
  if (paged) {
    int sh = 0;
    while ((1 << sh) < paged->page_rows) ++sh;
    prm.page_shift = static_cast<uint32_t>(sh);
    prm.page_mask = static_cast<uint32_t>(paged->page_rows - 1);
    prm.page_rows = static_cast<uint32_t>(paged->page_rows);
    prm.page_first = paged->first_offset;
  }
  // tensor maps per frame: Y + interleaved UV (NV12), or Y + U + V (I420)
  const int mpf = i420 ? 3 : 2;
  prm.sxmask = i420 ? ~31 : ~15;  // TMA box starts must be 16-byte aligned: SX0 (Y) and SX0/2 (U, V)
  const bool inline_maps = jobs.size() == 1 && mpf * nf <= 2 * kMaxInlineFrames;
  std::vector<CUtensorMap> maps(inline_maps ? 0 : mpf * nf);
  CUtensorMap* mp = inline_maps ? prm.tm : maps.data();
  for (size_t j = 0; j < jobs.size(); ++j)
    for (int64_t i = 0; i < nfj; ++i) {
      const fc_nv12_surface& sf = jobs[j].surfaces[jobs[j].frames[i]];
      const int64_t fi = static_cast<int64_t>(j) * nfj + i;
      st = tensor_map(sf.y, sf.pitch_y, H, g.BW, kChunkRows, &mp[mpf * fi]);
      if (i420) {
        if (st == FC_OK) st = tensor_map(sf.uv, sf.pitch_uv, H / 2, g.BW / 2, kChunkRows / 2, &mp[mpf * fi + 1]);
        if (st == FC_OK) st = tensor_map(sf.v, sf.pitch_uv, H / 2, g.BW / 2, kChunkRows / 2, &mp[mpf * fi + 2]);
      } else if (st == FC_OK) {
        st = tensor_map(sf.uv, sf.pitch_uv, H / 2, g.BW, kChunkRows / 2, &mp[mpf * fi + 1]);
      }
      if (st != FC_OK) return st;
    }
  if (dry) return FC_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  void* desc = nullptr;
  if (!inline_maps || paged) {
    // descriptor sections: [tensor maps | per-job token bases | page ids]
    const size_t mbytes = maps.size() * sizeof(CUtensorMap);
    const size_t tbytes = jobs.size() > 1 ? jobs.size() * sizeof(void*) : 0;
    const size_t pbytes = paged ? static_cast<size_t>(paged->num_pages) * sizeof(int32_t) : 0;
    const size_t bytes = mbytes + tbytes + pbytes;
    std::vector<uint8_t> host(bytes);
    std::memcpy(host.data(), maps.data(), mbytes);
    if (jobs.size() > 1)
      for (size_t j = 0; j < jobs.size(); ++j)
        std::memcpy(host.data() + mbytes + j * sizeof(void*), &jobs[j].tokens, sizeof(void*));
    if (paged) std::memcpy(host.data() + mbytes + tbytes, paged->page_ids, pbytes);
    cudaMemPool_t pool = descriptor_pool(dev);
    e = pool ? cudaMallocFromPoolAsync(&desc, bytes, pool, s) : cudaMallocAsync(&desc, bytes, s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync (launch descriptor)");
    // pageable source: returns once the bytes are staged, so `host` may die
    e = cudaMemcpyAsync(desc, host.data(), bytes, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) {
      cudaFreeAsync(desc, s);
      return cuda_fail(e, "descriptor upload");
    }
    if (!inline_maps) prm.tmg = reinterpret_cast<const CUtensorMap*>(desc);
    if (jobs.size() > 1) prm.tokj = reinterpret_cast<void* const*>(static_cast<uint8_t*>(desc) + mbytes);
    if (paged) prm.page_ids = reinterpret_cast<const int32_t*>(static_cast<uint8_t*>(desc) + mbytes + tbytes);
  }
  int grid = static_cast<int>(std::min<long long>(items, static_cast<long long>(occ) * nsm));
  // strip-synchronous work mapping (see the kernel): the CTAs of a strip walk
  // down the same frames side by side, so strip halos are L2 hits.  Per-launch
  // DRAM reads (single-pass ncu, round 2): c2 669 -> 404 MB, c3 1.70 -> 0.88 GB,
  // c4 1.04 -> 0.76 GB (746.5 MB of NV12), c5 1.75 GB -> ~0.8 GB, i.e. traffic
  // ~= the algorithmic bytes; kernel time c2 -0.2%, c3 +0.6%, c4 +2.3%, c5
  // +0.4% (the kernel is issue-bound, not DRAM-bound).  On for every launch.
  // FC_SMAP=0/1 forces it off/on (A/B runs).
  const char* smenv = std::getenv("FC_SMAP");
  if ((smenv ? std::atoi(smenv) != 0 : true) && grid >= g.nstrips) prm.smap = 1;
  unsigned long long* cta_t = nullptr;
  if (std::getenv("FC_CTA_TIMES") && cudaMalloc(&cta_t, 3 * sizeof(unsigned long long) * grid) == cudaSuccess) {
    cudaMemsetAsync(cta_t, 0, 3 * sizeof(unsigned long long) * grid, s);
    prm.cta_t = cta_t;
  }
  {
    // programmatic dependent launch: this launch's prologue (shared-memory
    // tables, barrier init) overlaps the previous launch's tail on the stream;
    // the kernel waits (griddepcontrol.wait) before any global access.
    // FC_PDL=0 turns it off (A/B runs).
    static const bool pdl = [] {
      const char* v = std::getenv("FC_PDL");
      return v ? std::atoi(v) != 0 : true;
    }();
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(kThreads);
    lc.dynamicSmemBytes = g.smem;
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = pdl ? 1 : 0;
    e = cudaLaunchKernelEx(&lc, fn, prm);
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  if (cta_t) {  // experiment: CTA lifetime distribution (start/end, ns from the first start)
    prm.cta_t = nullptr;
    std::vector<unsigned long long> t(3 * grid);
    cudaMemcpyAsync(t.data(), cta_t, t.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    cudaFree(cta_t);
    unsigned long long t0 = ~0ull, t1 = 0;
    for (int b = 0; b < grid; ++b) t0 = std::min(t0, t[3 * b]), t1 = std::max(t1, t[3 * b + 1]);
    std::vector<double> st(grid), en(grid);
    double busy = 0;
    for (int b = 0; b < grid; ++b) {
      st[b] = (t[3 * b] - t0) * 1e-3, en[b] = (t[3 * b + 1] - t0) * 1e-3;
      busy += en[b] - st[b];
    }
    std::vector<double> es = en, ss = st;
    std::sort(es.begin(), es.end());
    std::sort(ss.begin(), ss.end());
    std::fprintf(stderr,
                 "fc cta times (us): span %.1f | start max %.1f | end min %.1f p10 %.1f p50 %.1f p90 %.1f max %.1f | "
                 "mean lifetime / span %.3f\n",
                 (t1 - t0) * 1e-3, ss.back(), es.front(), es[grid / 10], es[grid / 2], es[grid * 9 / 10], es.back(),
                 busy / grid / ((t1 - t0) * 1e-3));
    if (const char* f = std::getenv("FC_CTA_TIMES_FILE")) {
      if (FILE* fp = std::fopen(f, "a")) {
        for (int b = 0; b < grid; ++b) std::fprintf(fp, "%d %llu %.2f %.2f\n", b, t[3 * b + 2], st[b], en[b]);
        std::fclose(fp);
      }
    }
  }
  if (desc) cudaFreeAsync(desc, s);
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  last_kernel() = FC_KERNEL_MMA;
  return FC_OK;
}

// Token buffers are written with 8-byte (fp32 pairs), 4-byte (bf16 pairs) or
// 2-byte (u8 pairs) stores: a misaligned view would fault the context, so
// it is rejected up front.
static bool tokens_aligned(const void* p, fc_token_dtype td) {
  const uintptr_t m = td == FC_TOKENS_F32 ? 7 : td == FC_TOKENS_BF16 ? 3 : 1;
  return (reinterpret_cast<uintptr_t>(p) & m) == 0;
}

static fc_status preprocess_impl(const fc_plan_t* Pc, int32_t rank, const fc_nv12_surface* surfaces,
                                 int64_t num_surfaces, void* tokens, int64_t grid_thw[3], void* stream,
                                 uint8_t* dbg_src, uint8_t* dbg_rs, const fc_paged_tokens* paged = nullptr,
                                 bool colsplit = false) {
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
  if (!tokens && !paged) return fail(FC_ERR_INVALID_ARG, "tokens is NULL");
  if (!tokens_aligned(paged ? paged->pool : tokens, P->cfg.token_dtype))
    return fail(FC_ERR_UNSUPPORTED, "token buffer not aligned to its store width (8 B fp32, 4 B bf16, 2 B u8)");
  if (paged) {  // the page table must hold the write (SPEC write_chunk: CapacityError)
    const fc_rank_plan& rp = P->ranks[rank].p;
    const int64_t rows = rp.row_end - rp.row_begin;
    if (!paged->pool || !paged->page_ids || paged->page_rows <= 0 || (paged->page_rows & (paged->page_rows - 1)))
      return fail(FC_ERR_INVALID_ARG, "paged output: pool/page_ids NULL or page_rows not a power of two");
    if (paged->first_offset < 0 || paged->first_offset >= paged->page_rows)
      return fail(FC_ERR_INVALID_ARG, "paged output: first_offset outside [0, page_rows)");
    if (paged->num_pages < (paged->first_offset + rows + paged->page_rows - 1) / paged->page_rows)
      return fail(FC_ERR_INVALID_ARG, "paged output: not enough pages for the rank's rows");
    for (int32_t i = 0; i < paged->num_pages; ++i)
      if (paged->page_ids[i] < 0 || paged->page_ids[i] >= paged->pool_pages ||
          static_cast<int64_t>(paged->page_ids[i] + 1) * paged->page_rows > UINT32_MAX)
        return fail(FC_ERR_INVALID_ARG, "paged output: page id outside the pool");
  }
  jobs[0].surfaces = surfaces;
  jobs[0].tokens = tokens;
  if (colsplit && kCols % P->world != 0)
    return fail(FC_ERR_UNSUPPORTED, "column-split output: world_size must divide 1176");
  return launch_jobs(P, jobs, stream, dbg_src, dbg_rs, paged, colsplit);
}

}  // namespace fc

using namespace fc;

extern "C" {

fc_status fc_preprocess(const fc_plan_t* plan, int32_t rank, const fc_nv12_surface* surfaces,
                        int64_t num_surfaces, void* tokens, int64_t grid_thw[3], void* stream) {
  NvtxRange nvtx("fc_preprocess");
  return preprocess_impl(plan, rank, surfaces, num_surfaces, tokens, grid_thw, stream, nullptr, nullptr);
}

fc_status fc_submit(const fc_video_meta* meta, const fc_model_cfg* cfg, int32_t rank, const fc_nv12_surface* surfaces,
                    int64_t num_surfaces, void* tokens, void* stream, fc_plan_t** plan_out) {
  NvtxRange nvtx("fc_submit");
  if (!plan_out) return fail(FC_ERR_INVALID_ARG, "plan_out is NULL");
  *plan_out = nullptr;
  fc_plan_t* P = nullptr;
  fc_status st = fc_plan(meta, cfg, &P);
  if (st != FC_OK) return st;
  st = preprocess_impl(P, rank, surfaces, num_surfaces, tokens, nullptr, stream, nullptr, nullptr);
  if (st != FC_OK) {
    fc_plan_destroy(P);
    return st;
  }
  *plan_out = P;
  return FC_OK;
}

fc_status fc_preprocess_colsplit(const fc_plan_t* plan, int32_t rank, const fc_nv12_surface* surfaces,
                                 int64_t num_surfaces, float* blocks, int64_t grid_thw[3], void* stream) {
  return preprocess_impl(plan, rank, surfaces, num_surfaces, blocks, grid_thw, stream, nullptr, nullptr, nullptr, true);
}

fc_status fc_preprocess_paged(const fc_plan_t* plan, int32_t rank, const fc_nv12_surface* surfaces,
                              int64_t num_surfaces, const fc_paged_tokens* out, int64_t grid_thw[3], void* stream) {
  if (!out) return fail(FC_ERR_INVALID_ARG, "paged descriptor is NULL");
  return preprocess_impl(plan, rank, surfaces, num_surfaces, nullptr, grid_thw, stream, nullptr, nullptr, out);
}

fc_status fc_preprocess_debug(const fc_plan_t* plan, int32_t rank, const fc_nv12_surface* surfaces,
                              int64_t num_surfaces, void* tokens, int64_t grid_thw[3], void* stream,
                              uint8_t* rgb_src, uint8_t* rgb_resized) {
  return preprocess_impl(plan, rank, surfaces, num_surfaces, tokens, grid_thw, stream, rgb_src, rgb_resized);
}

fc_status fc_preprocess_batch(const fc_plan_t* const* plans, const int32_t* ranks, int32_t count,
                              const fc_nv12_surface* const* surfaces, const int64_t* num_surfaces,
                              void* const* tokens, void* stream) {
  NvtxRange nvtx("fc_preprocess_batch");
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
    if (!jobs[i].frames.empty() && !tokens_aligned(tokens[i], jp[i]->cfg.token_dtype))
      return fail(FC_ERR_UNSUPPORTED, "batch: token buffer not aligned to its store width");
    jobs[i].surfaces = surfaces[i];
    jobs[i].tokens = tokens[i];
  }
  auto same = [&](int a, int b) {
    const fc_plan_s &A = *jp[a], &B = *jp[b];
    return A.meta.width == B.meta.width && A.meta.height == B.meta.height && A.w2 == B.w2 && A.h2 == B.h2 &&
           A.cfg.token_dtype == B.cfg.token_dtype && A.cfg.color == B.cfg.color && A.lut_dev == B.lut_dev &&
           A.cfg.surface_format == B.cfg.surface_format &&
           jobs[a].frames.size() == jobs[b].frames.size();
  };
  // groups; every group is validated (dry run) before the first launch, so an
  // error leaves nothing enqueued (fc.h: no partial effects)
  std::vector<std::pair<int32_t, std::vector<Job>>> groups;
  for (int32_t i = 0; i < count;) {
    if (jobs[i].frames.empty()) {
      ++i;
      continue;
    }
    int32_t j = i;
    std::vector<Job> group;
    while (j < count && (jobs[j].frames.empty() || same(i, j))) {
      if (!jobs[j].frames.empty()) group.push_back(jobs[j]);
      ++j;
    }
    groups.emplace_back(i, std::move(group));
    i = j;
  }
  for (auto& g : groups) {
    fc_status st = launch_jobs(jp[g.first], g.second, stream, nullptr, nullptr, nullptr, false, true);
    if (st != FC_OK) return st;
  }
  for (auto& g : groups) {
    fc_status st = launch_jobs(jp[g.first], g.second, stream, nullptr, nullptr);
    if (st != FC_OK) return st;
  }
  return FC_OK;
}

uint64_t fc_kernel_launches(void) { return launch_counter().load(std::memory_order_relaxed); }

int32_t fc_last_kernel(void) { return last_kernel(); }

void fc_plan_destroy(fc_plan_t* P) {
  // device tables belong to the process-wide cache (shared by equal shapes)
  delete P;
}

}  // extern "C"
