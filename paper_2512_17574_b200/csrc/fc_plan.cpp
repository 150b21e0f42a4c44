// fc_plan.cpp -- host planner of libfc.so: the planning half of Alg. 1
// plus the per-plan coefficient / normalisation
// tables the fused kernel consumes.  Compiled with -ffp-contract=off: every
// f64 / f32 operation below must round exactly as written (R2, R4, R5).
//
// Readings:
//   R1 sampling      = HF Qwen2VLVideoProcessor.sample_frames (P:319 silent)
//   R2 resize target = HF smart_resize, Python round-half-even
//   R4 resize        = Pillow ImagingResample BICUBIC, 22-bit ints, H then V
//   R5 normalise     = f32((f64(v)*rescale)) then f32 (x-mean)/std
//   R21 backends     = PIL (R4, R5) or torchvision on CPU (torch's uint8 AA
//                      bicubic precision rule, HF's fused normalisation)
//   R8 partition     = contiguous GOP ranges, method b, exact DP
#include <algorithm>
#include <climits>
#include <cmath>
#include <map>
#include <tuple>
#include <memory>
#include <cstring>
#include <limits>
#include <new>

#include "fc_internal.h"

namespace fc {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }
fc_status fail(fc_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

// ---------------------------------------------------------------- R4 tables
// Pillow's bicubic kernel, a = -0.5 (libImaging/Resample.c bicubic_filter).
static double bicubic(double x) {
  const double a = -0.5;
  if (x < 0.0) x = -x;
  if (x < 1.0) return ((a + 2.0) * x - (a + 3.0)) * x * x + 1;
  if (x < 2.0) return (((x - 5) * x + 8) * x - 4) * a;
  return 0.0;
}

// Pillow precompute_coeffs + normalize_coeffs_8bpc for in -> out (R4).  The
// torchvision backend (R21) keeps the windows and double weights and rounds
// them at torch's int16 precision p instead of 22 bits; the table holds
// round(w*2^p) << (22 - p), so the kernels' 22-bit arithmetic,
// clamp((2^21 + sum px*iw) >> 22), is exactly torch's clamp((2^(p-1) + sum
// px*round(w*2^p)) >> p).
fc_status build_axis(int in, int out, int backend, AxisTable* t) {
  t->in = in;
  t->out = out;
  const double scale = static_cast<double>(in) / static_cast<double>(out);
  const double filterscale = std::max(scale, 1.0);
  const double support = 2.0 * filterscale;
  const int ksize = static_cast<int>(std::ceil(support)) * 2 + 1;
  t->ksize = ksize;
  t->xmin.assign(out, 0);
  t->cnt.assign(out, 0);
  t->iw.assign(static_cast<size_t>(out) * ksize, 0);
  std::vector<double> kall(static_cast<size_t>(out) * ksize, 0.0);  // normalised weights of every output
  double wmax = 0.0;
  int max_cnt = 0;
  for (int o = 0; o < out; ++o) {
    double* k = &kall[static_cast<size_t>(o) * ksize];
    const double center = (o + 0.5) * scale;
    double ww = 0.0;
    const double ss = 1.0 / filterscale;
    int xmin = static_cast<int>(center - support + 0.5);
    if (xmin < 0) xmin = 0;
    int xmax = static_cast<int>(center + support + 0.5);
    if (xmax > in) xmax = in;
    xmax -= xmin;
    for (int x = 0; x < xmax; ++x) {
      const double w = bicubic((x + xmin - center + 0.5) * ss);
      k[x] = w;
      ww += w;
    }
    for (int x = 0; x < xmax; ++x)
      if (ww != 0.0) k[x] /= ww;
    for (int x = 0; x < xmax; ++x) wmax = std::max(wmax, k[x]);
    t->xmin[o] = xmin;
    t->cnt[o] = xmax;
    max_cnt = std::max(max_cnt, xmax);
  }
  t->max_cnt = max_cnt;
  int prec = kPrecisionBits;
  if (backend == FC_BACKEND_TORCHVISION)  // torch: the largest p < 22 keeping every weight an int16
    for (prec = 0; prec < 22; ++prec)
      if (static_cast<int>(0.5 + wmax * (1 << (prec + 1))) >= (1 << 15)) break;
  t->prec = prec;
  for (int o = 0; o < out; ++o)
    for (int x = 0; x < t->cnt[o]; ++x) {
      const double w = kall[static_cast<size_t>(o) * ksize + x];
      const int32_t q = static_cast<int32_t>(w < 0 ? -0.5 + w * (1 << prec) : 0.5 + w * (1 << prec));
      t->iw[static_cast<size_t>(o) * ksize + x] = static_cast<int32_t>(static_cast<uint32_t>(q) << (kPrecisionBits - prec));
    }
  // the kernels split each weight into three bytes (the mma.sync kernel: two
  // unsigned low bytes and a signed high byte), so |iw| < 2^23 is required
  for (int o = 0; o < out; ++o)
    for (int kk = 0; kk < t->cnt[o]; ++kk) {
      const int32_t hi = t->iw[static_cast<size_t>(o) * ksize + kk] >> 16;
      if (hi < -128 || hi > 127) return fail(FC_ERR_UNSUPPORTED, "resize weight out of byte-plane range");
    }
  return FC_OK;
}

// Axis tables depend only on (in, out): requests of one resolution share them
// (a serving process sees few distinct shapes).  Bounded; evicted tables stay
// alive while a plan holds them.
fc_status axis_cached(int in, int out, int backend, std::shared_ptr<const AxisTable>* t) {
  static std::mutex mu;
  static auto* cache = new std::map<std::tuple<int, int, int>, std::shared_ptr<const AxisTable>>();  // never freed
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache->find({in, out, backend});
    if (it != cache->end()) {
      *t = it->second;
      return FC_OK;
    }
  }
  auto a = std::make_shared<AxisTable>();
  fc_status st = build_axis(in, out, backend, a.get());
  if (st != FC_OK) return st;
  std::lock_guard<std::mutex> lk(mu);
  if (cache->size() >= 256) cache->clear();
  (*cache)[{in, out, backend}] = a;
  *t = a;
  return FC_OK;
}

// ---------------------------------------------------------------- R1 sampling
static fc_status sample(const fc_video_meta& m, const fc_model_cfg& c, std::vector<int64_t>* idx) {
  const int64_t N = m.num_frames;
  const int tps = c.temporal_patch_size;
  idx->clear();
  if (c.sampling == FC_SAMPLE_EXPLICIT) {
    if (!c.explicit_indices || c.num_explicit <= 0)
      return fail(FC_ERR_EMPTY_SELECTION, "explicit sampling with an empty list");
    for (int64_t i = 0; i < c.num_explicit; ++i) {
      const int64_t v = c.explicit_indices[i];
      if (v < 0 || v >= N) return fail(FC_ERR_INVALID_ARG, "explicit index out of range");
      if (i && v <= c.explicit_indices[i - 1])
        return fail(FC_ERR_INVALID_ARG, "explicit indices must be strictly increasing");
      idx->push_back(v);
    }
    return FC_OK;
  }
  int64_t n;
  if (c.num_frames > 0) {
    // HF: round(num_frames / tps) * tps  (Python round = half to even)
    n = static_cast<int64_t>(std::nearbyint(static_cast<double>(c.num_frames) / tps)) * tps;
  } else {
    if (!(c.sample_fps > 0)) return fail(FC_ERR_INVALID_ARG, "sample_fps must be > 0");
    const double fps_src = static_cast<double>(m.fps.num) / static_cast<double>(m.fps.den);
    const double maxf = std::floor(static_cast<double>(std::min<int64_t>(c.max_frames, N)) / tps) * tps;
    double x = static_cast<double>(N) / fps_src * c.sample_fps;
    x = std::max(x, static_cast<double>(c.min_frames));
    x = std::min(std::min(x, maxf), static_cast<double>(N));
    n = static_cast<int64_t>(std::floor(x / tps)) * tps;
  }
  if (n <= 0 || n > N)
    return fail(FC_ERR_EMPTY_SELECTION, "sampling selects n=" + std::to_string(n) + " of N=" + std::to_string(N));
  idx->resize(n);
  if (c.sampling == FC_SAMPLE_LINSPACE) {
    for (int64_t i = 0; i < n; ++i) {
      if (n == 1) { (*idx)[i] = 0; continue; }
      const int64_t num = i * (N - 1), den = n - 1;
      int64_t q = num / den;
      const int64_t r = num % den;
      if (2 * r > den || (2 * r == den && (q & 1))) ++q;
      (*idx)[i] = q;
    }
  } else if (c.sampling == FC_SAMPLE_FPS_STRIDE) {
    for (int64_t i = 0; i < n; ++i) (*idx)[i] = (i * N) / n;
  } else {
    return fail(FC_ERR_UNSUPPORTED, "unknown sampling mode");
  }
  return FC_OK;
}

// ---------------------------------------------------------------- R2 resize
static fc_status smart_resize(int64_t H, int64_t W, const fc_model_cfg& c, int64_t n, int32_t* h2,
                              int32_t* w2) {
  const int factor = c.patch_size * c.merge_size;
  if (c.resized_height > 0 || c.resized_width > 0) {
    if (c.resized_height <= 0 || c.resized_width <= 0 || c.resized_height % factor || c.resized_width % factor)
      return fail(FC_ERR_INVALID_ARG, "resized_height/width must both be positive multiples of 28");
    *h2 = c.resized_height;
    *w2 = c.resized_width;
    return FC_OK;
  }
  if (static_cast<double>(std::max(H, W)) / static_cast<double>(std::min(H, W)) > 200.0)
    return fail(FC_ERR_ASPECT_RATIO, "absolute aspect ratio must be <= 200");
  double min_pixels = static_cast<double>(c.min_pixels);
  double max_pixels = static_cast<double>(c.max_pixels);
  if (c.total_pixels > 0) {  // qwen-vl-utils total budget (R2 variant)
    max_pixels = std::max(std::min(max_pixels, c.total_pixels / static_cast<double>(n) * c.temporal_patch_size),
                          std::floor(min_pixels * 1.05));
  }
  const double f = factor;
  double h_bar = std::nearbyint(static_cast<double>(H) / f) * f;
  double w_bar = std::nearbyint(static_cast<double>(W) / f) * f;
  if (h_bar * w_bar > max_pixels) {
    const double beta = std::sqrt(static_cast<double>(H * W) / max_pixels);
    h_bar = std::max(f, std::floor(static_cast<double>(H) / beta / f) * f);
    w_bar = std::max(f, std::floor(static_cast<double>(W) / beta / f) * f);
  } else if (h_bar * w_bar < min_pixels) {
    const double beta = std::sqrt(min_pixels / static_cast<double>(H * W));
    h_bar = std::ceil(static_cast<double>(H) * beta / f) * f;
    w_bar = std::ceil(static_cast<double>(W) * beta / f) * f;
  }
  if (h_bar < f || w_bar < f || h_bar > 1 << 20 || w_bar > 1 << 20)
    return fail(FC_ERR_UNSUPPORTED, "resized size out of range");
  *h2 = static_cast<int32_t>(h_bar);
  *w2 = static_cast<int32_t>(w_bar);
  return FC_OK;
}

// ---------------------------------------------------------------- R8 partition
namespace {
struct Seg {
  int64_t start, end, pairs, pad;
  bool tail;
};

// Method b applied to one rank taking GOPs [b, b2) with `start` sampled
// positions already consumed: returns false if the rank would be empty.
bool rank_step(const std::vector<int64_t>& a, int64_t n, int G, int b2, int64_t start, Seg* s) {
  int64_t end = (b2 == G) ? n : std::max(a[b2], start);
  int64_t cnt = end - start;
  if (cnt <= 0) return false;
  s->tail = false;
  if ((cnt % kTps) && end < n) {  // method b: take the next sampled frame
    end += kTps - cnt % kTps;
    cnt = end - start;
    s->tail = true;
  }
  s->pad = (cnt % kTps) ? (kTps - cnt % kTps) : 0;  // only reachable when end == n
  s->start = start;
  s->end = end;
  s->pairs = (cnt + s->pad) / kTps;
  return true;
}

struct Cost2 {
  int64_t enc, sq;  // lexicographic: -encoder pairs, sum of pairs^2
  bool operator<(const Cost2& o) const { return enc != o.enc ? enc < o.enc : sq < o.sq; }
};
}  // namespace

static fc_status partition(fc_plan_s* P) {
  const int G = static_cast<int>(P->gop_start.size());
  const int W = P->world;
  const int64_t n = P->n;
  const int64_t N = P->meta.num_frames;
  // per-GOP sampled counts and prefix positions a[b]
  std::vector<int64_t> a(G + 1, 0);
  {
    int g = 0;
    std::vector<int64_t> s(G, 0);
    for (int64_t f : P->sampled) {
      while (g + 1 < G && P->gop_start[g + 1] <= f) ++g;
      s[g]++;
    }
    for (int b = 0; b < G; ++b) a[b + 1] = a[b] + s[b];
  }
  (void)N;
  // state (b, c): next rank starts at sampled position a[b] + c, c in {0,1}
  const int64_t INF = std::numeric_limits<int64_t>::max() / 4;
  // ---- phase 1: minimise the maximum per-rank pairs
  std::vector<int64_t> F((G + 1) * 2, INF), NF((G + 1) * 2, INF);
  F[0] = 0;
  int64_t best = INF;
  for (int r = 0; r < W; ++r) {
    std::fill(NF.begin(), NF.end(), INF);
    for (int b = 0; b < G; ++b)
      for (int c = 0; c < 2; ++c) {
        const int64_t cur = F[b * 2 + c];
        if (cur >= INF) continue;
        const int64_t start = a[b] + c;
        for (int b2 = b + 1; b2 <= G; ++b2) {
          Seg s;
          if (!rank_step(a, n, G, b2, start, &s)) continue;
          if (s.pairs > best) break;  // pairs never decrease as b2 grows: no later b2 can beat best
          const int64_t v = std::max(cur, s.pairs);
          if (s.end == n) {
            best = std::min(best, v);
          } else {
            const int c2 = static_cast<int>(s.end - a[b2]);
            NF[b2 * 2 + c2] = std::min(NF[b2 * 2 + c2], v);
          }
        }
      }
    F.swap(NF);
  }
  if (best >= INF) return fail(FC_ERR_INVALID_ARG, "no valid GOP partition (internal)");
  const int64_t cap = best;
  // ---- phase 2: under the cap, maximise the encoder rank's pairs, then
  //      minimise sum of pairs^2 (balance); ties keep the first found.
  struct Node {
    Cost2 cost;
    int pb, pc;  // predecessor state
    bool valid;
  };
  const int e = P->cfg.encoder_rank;
  std::vector<std::vector<Node>> T(W + 1, std::vector<Node>((G + 1) * 2, Node{{0, 0}, -1, -1, false}));
  T[0][0] = Node{{0, 0}, -1, -1, true};
  Cost2 best2{INF, INF};
  int best_r = -1, best_b = -1, best_c = -1, best_b2 = -1;
  for (int r = 0; r < W; ++r)
    for (int b = 0; b < G; ++b)
      for (int c = 0; c < 2; ++c) {
        const Node& cur = T[r][b * 2 + c];
        if (!cur.valid) continue;
        const int64_t start = a[b] + c;
        for (int b2 = b + 1; b2 <= G; ++b2) {
          Seg s;
          if (!rank_step(a, n, G, b2, start, &s)) continue;
          if (s.pairs > cap) break;  // pairs never decrease as b2 grows
          Cost2 nc{cur.cost.enc - (r == e ? s.pairs : 0), cur.cost.sq + s.pairs * s.pairs};
          if (s.end == n) {
            if (nc < best2) {
              best2 = nc;
              best_r = r;
              best_b = b;
              best_c = c;
              best_b2 = b2;
            }
          } else {
            const int c2 = static_cast<int>(s.end - a[b2]);
            Node& nx = T[r + 1][b2 * 2 + c2];
            if (!nx.valid || nc < nx.cost) nx = Node{nc, b * 2 + c, 0, true};
          }
        }
      }
  if (best_r < 0) return fail(FC_ERR_INVALID_ARG, "no valid GOP partition under cap (internal)");
  // backtrack the boundary states
  std::vector<std::pair<int, int>> states;  // (b, c) at the start of each rank
  std::vector<int> ends;                    // b2 of each rank
  {
    int r = best_r, st = best_b * 2 + best_c, b2 = best_b2;
    while (r >= 0) {
      states.push_back({st / 2, st % 2});
      ends.push_back(b2);
      const Node& nd = T[r][st];
      b2 = st / 2;
      st = nd.pb;
      --r;
    }
    std::reverse(states.begin(), states.end());
    std::reverse(ends.begin(), ends.end());
  }
  const int used = static_cast<int>(states.size());
  P->ranks.assign(W, RankPlan{});
  P->ranks_used = used;
  int64_t row = 0;
  const int64_t rows_per_pair = P->gh * P->gw;
  auto gop_of = [&](int64_t f) {
    return static_cast<int64_t>(std::upper_bound(P->gop_start.begin(), P->gop_start.end(), f) -
                                P->gop_start.begin()) - 1;
  };
  for (int r = 0; r < W; ++r) {
    fc_rank_plan& rp = P->ranks[r].p;
    if (r >= used) {
      rp = fc_rank_plan{G, G, -1, -1, n, 0, 0, row, row, 0};
      continue;
    }
    Seg s;
    const int64_t start = a[states[r].first] + states[r].second;
    rank_step(a, n, G, ends[r], start, &s);
    const int64_t body_end = s.tail ? s.end - 1 : s.end;
    rp.sampled_begin = s.start;
    rp.sampled_count = s.end - s.start;
    rp.pad_frames = s.pad;
    rp.gop_begin = gop_of(P->sampled[s.start]);
    rp.gop_end = gop_of(P->sampled[body_end - 1]) + 1;
    rp.tail_frame = s.tail ? P->sampled[s.end - 1] : -1;
    rp.tail_gop = s.tail ? gop_of(rp.tail_frame) : -1;
    rp.row_begin = row;
    row += s.pairs * rows_per_pair;
    rp.row_end = row;
    // frames NVDEC would decode: keyframe .. last target, per GOP
    int64_t est = 0;
    for (int64_t i = s.start; i < body_end;) {
      const int64_t g = gop_of(P->sampled[i]);
      int64_t j = i;
      while (j + 1 < body_end && gop_of(P->sampled[j + 1]) == g) ++j;
      est += P->sampled[j] - P->gop_start[g] + 1;
      i = j + 1;
    }
    if (s.tail) est += rp.tail_frame - P->gop_start[rp.tail_gop] + 1;
    rp.est_decode_frames = est;
  }
  return FC_OK;
}

}  // namespace fc

using namespace fc;

extern "C" {

void fc_model_cfg_default(fc_model_cfg* c) {
  if (!c) return;
  std::memset(c, 0, sizeof(*c));
  c->patch_size = 14;
  c->temporal_patch_size = 2;
  c->merge_size = 2;
  c->min_pixels = 128 * 28 * 28;
  c->max_pixels = 768 * 28 * 28;
  c->total_pixels = 0;
  c->sampling = FC_SAMPLE_FPS_STRIDE;
  c->sample_fps = 2.0;
  c->num_frames = 0;
  c->min_frames = 4;
  c->max_frames = 768;
  c->explicit_indices = nullptr;
  c->num_explicit = 0;
  c->resized_height = 0;
  c->resized_width = 0;
  const float mean[3] = {0.48145466f, 0.4578275f, 0.40821073f};
  const float stdv[3] = {0.26862954f, 0.26130258f, 0.27577711f};
  for (int i = 0; i < 3; ++i) {
    c->image_mean[i] = mean[i];
    c->image_std[i] = stdv[i];
  }
  c->rescale_factor = 1.0 / 255.0;
  c->world_size = 1;
  c->encoder_rank = 0;
  c->backend = FC_BACKEND_PIL;
}

fc_status fc_plan(const fc_video_meta* meta, const fc_model_cfg* cfg, fc_plan_t** out) {
  NvtxRange nvtx("fc_plan");
  if (!out) return fail(FC_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (!meta || !cfg) return fail(FC_ERR_INVALID_ARG, "meta/cfg is NULL");
  const fc_video_meta& m = *meta;
  if (m.width < 2 || m.height < 2) return fail(FC_ERR_INVALID_ARG, "width/height must be >= 2");
  if ((m.width & 1) || (m.height & 1)) return fail(FC_ERR_UNSUPPORTED, "NV12 needs even width and height");
  if (m.width > (1 << 16) || m.height > (1 << 16)) return fail(FC_ERR_UNSUPPORTED, "frame too large");
  if (m.num_frames < 1) return fail(FC_ERR_INVALID_ARG, "num_frames must be >= 1");
  if (m.fps.num <= 0 || m.fps.den <= 0) return fail(FC_ERR_INVALID_ARG, "fps must be a positive rational");
  if (m.num_gops < 1 || !m.gop_start) return fail(FC_ERR_INVALID_ARG, "need >= 1 GOP");
  if (m.gop_start[0] != 0) return fail(FC_ERR_INVALID_ARG, "gop_start[0] must be 0");
  for (int64_t g = 0; g < m.num_gops; ++g) {
    if (m.gop_start[g] >= m.num_frames) return fail(FC_ERR_INVALID_ARG, "gop_start beyond num_frames");
    if (g && m.gop_start[g] <= m.gop_start[g - 1])
      return fail(FC_ERR_INVALID_ARG, "gop_start must be strictly increasing");
  }
  const fc_model_cfg& c = *cfg;
  if (c.patch_size != kPatch || c.temporal_patch_size != kTps || c.merge_size != kMerge)
    return fail(FC_ERR_UNSUPPORTED, "only patch 14, temporal patch 2, merge 2 are supported");
  if (c.world_size < 1 || c.world_size > 1024) return fail(FC_ERR_INVALID_ARG, "world_size out of range [1, 1024]");
  if (c.encoder_rank < 0 || c.encoder_rank >= c.world_size)
    return fail(FC_ERR_RANK, "encoder_rank outside [0, world_size)");
  if (c.min_frames < 0 || c.max_frames < 1) return fail(FC_ERR_INVALID_ARG, "bad min/max frames");
  if (!(c.rescale_factor > 0)) return fail(FC_ERR_INVALID_ARG, "rescale_factor must be > 0");
  for (int i = 0; i < 3; ++i)
    if (!(c.image_std[i] != 0.0f)) return fail(FC_ERR_INVALID_ARG, "image_std must be non-zero");
  if (c.token_dtype != FC_TOKENS_F32 && c.token_dtype != FC_TOKENS_BF16 && c.token_dtype != FC_TOKENS_U8)
    return fail(FC_ERR_UNSUPPORTED, "unknown token_dtype");
  if (c.color < FC_COLOR_BT601_LIMITED || c.color > FC_COLOR_BT709_FULL)
    return fail(FC_ERR_UNSUPPORTED, "unknown color matrix");
  if (c.backend != FC_BACKEND_PIL && c.backend != FC_BACKEND_TORCHVISION)
    return fail(FC_ERR_UNSUPPORTED, "unknown backend");
  if (c.surface_format != FC_SURFACE_NV12 && c.surface_format != FC_SURFACE_I420)
    return fail(FC_ERR_UNSUPPORTED, "unknown surface format");

  fc_plan_s* P = new (std::nothrow) fc_plan_s();
  if (!P) return fail(FC_ERR_OOM, "plan allocation failed");
  P->meta = m;
  P->gop_start.assign(m.gop_start, m.gop_start + m.num_gops);
  P->meta.gop_start = P->gop_start.data();
  P->cfg = c;
  P->cfg.explicit_indices = nullptr;  // copied into `sampled`, never retained
  P->world = c.world_size;
  fc_status st = sample(m, c, &P->sampled);
  if (st == FC_OK) {
    P->n = static_cast<int64_t>(P->sampled.size());
    st = smart_resize(m.height, m.width, c, P->n, &P->h2, &P->w2);
  }
  if (st == FC_OK) {
    P->gt = (P->n + kTps - 1) / kTps;
    P->gh = P->h2 / kPatch;
    P->gw = P->w2 / kPatch;
    P->sampled_fps = static_cast<double>(P->n) / static_cast<double>(m.num_frames) *
                     (static_cast<double>(m.fps.num) / static_cast<double>(m.fps.den));
    P->second_per_grid = kTps / P->sampled_fps;
    try {  // the DP tables are O(W * G): no exception may cross the C ABI
      st = partition(P);
    } catch (const std::bad_alloc&) {
      st = fail(FC_ERR_OOM, "partition tables: host allocation failed");
    }
  }
  if (st == FC_OK) st = axis_cached(m.width, P->w2, c.backend, &P->th);
  if (st == FC_OK) st = axis_cached(m.height, P->h2, c.backend, &P->tv);
  if (st == FC_OK) {
    P->lut.resize(3 * 256);
    for (int ch = 0; ch < 3; ++ch)
      for (int v = 0; v < 256; ++v) {
        if (c.backend == FC_BACKEND_TORCHVISION) {  // R21: HF's fused rescale + normalise, float32
          const float inv = static_cast<float>(1.0 / c.rescale_factor);
          const float m2 = c.image_mean[ch] * inv, s2 = c.image_std[ch] * inv;
          const float d = static_cast<float>(v) - m2;
          P->lut[ch * 256 + v] = d / s2;
        } else {  // R5
          const float x = static_cast<float>(static_cast<double>(v) * c.rescale_factor);
          const float d = x - c.image_mean[ch];
          P->lut[ch * 256 + v] = d / c.image_std[ch];
        }
      }
    // the table the kernel stores from: fp32 bits, or (R16) the bf16 bits of
    // the fp32 value rounded to nearest-even, zero-extended (finite values)
    P->lut_dev.resize(3 * 256);
    for (int i = 0; i < 3 * 256; ++i) {
      uint32_t b;
      std::memcpy(&b, &P->lut[i], 4);
      P->lut_dev[i] = c.token_dtype == FC_TOKENS_BF16 ? (b + 0x7FFFu + ((b >> 16) & 1u)) >> 16 : b;
    }
  }
  if (st != FC_OK) {
    delete P;
    return st;
  }
  *out = P;
  return FC_OK;
}

fc_status fc_plan_info_get(const fc_plan_t* P, fc_plan_info* info) {
  if (!P || !info) return fail(FC_ERR_INVALID_ARG, "plan/info is NULL");
  info->grid_thw[0] = P->gt;
  info->grid_thw[1] = P->gh;
  info->grid_thw[2] = P->gw;
  info->resized_h = P->h2;
  info->resized_w = P->w2;
  info->num_sampled = P->n;
  info->pad_frames = (kTps - P->n % kTps) % kTps;
  info->token_rows = P->gt * P->gh * P->gw;
  info->token_cols = kCols;
  info->sampled_fps = P->sampled_fps;
  info->second_per_grid = P->second_per_grid;
  info->ranks_used = P->ranks_used;
  info->world_size = P->world;
  info->max_taps_h = P->th->max_cnt;
  info->max_taps_v = P->tv->max_cnt;
  return FC_OK;
}

fc_status fc_plan_sampled_indices(const fc_plan_t* P, int64_t* out) {
  if (!P || !out) return fail(FC_ERR_INVALID_ARG, "plan/out is NULL");
  std::memcpy(out, P->sampled.data(), sizeof(int64_t) * P->sampled.size());
  return FC_OK;
}

fc_status fc_plan_rank(const fc_plan_t* P, int32_t rank, fc_rank_plan* out) {
  if (!P || !out) return fail(FC_ERR_INVALID_ARG, "plan/out is NULL");
  if (rank < 0 || rank >= P->world) return fail(FC_ERR_RANK, "rank outside [0, world_size)");
  *out = P->ranks[rank].p;
  return FC_OK;
}

fc_status fc_assign_requests(const int64_t* pairs, int32_t n, int32_t world, int32_t* rank_of) {
  if (n < 0 || world < 1 || (n > 0 && (!pairs || !rank_of))) return fail(FC_ERR_INVALID_ARG, "assign_requests arguments");
  std::vector<int32_t> order(static_cast<size_t>(n));
  for (int32_t i = 0; i < n; ++i) {
    if (pairs[i] < 0) return fail(FC_ERR_INVALID_ARG, "negative pair count");
    order[static_cast<size_t>(i)] = i;
  }
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return pairs[a] > pairs[b]; });
  std::vector<int64_t> load(static_cast<size_t>(world), 0);
  for (int32_t i : order) {
    int32_t best = 0;
    for (int32_t r = 1; r < world; ++r)
      if (load[static_cast<size_t>(r)] < load[static_cast<size_t>(best)]) best = r;
    rank_of[i] = best;
    load[static_cast<size_t>(best)] += pairs[i];
  }
  return FC_OK;
}

const char* fc_status_string(fc_status s) {
  switch (s) {
    case FC_OK: return "FC_OK";
    case FC_ERR_INVALID_ARG: return "FC_ERR_INVALID_ARG";
    case FC_ERR_EMPTY_SELECTION: return "FC_ERR_EMPTY_SELECTION";
    case FC_ERR_ASPECT_RATIO: return "FC_ERR_ASPECT_RATIO";
    case FC_ERR_UNSUPPORTED: return "FC_ERR_UNSUPPORTED";
    case FC_ERR_MISSING_SURFACE: return "FC_ERR_MISSING_SURFACE";
    case FC_ERR_RANK: return "FC_ERR_RANK";
    case FC_ERR_OOM: return "FC_ERR_OOM";
    case FC_ERR_CUDA: return "FC_ERR_CUDA";
    case FC_ERR_NCCL: return "FC_ERR_NCCL";
    case FC_ERR_OUT_OF_PAGES: return "FC_ERR_OUT_OF_PAGES";
  }
  return "FC_ERR_UNKNOWN";
}

const char* fc_last_error(void) { return g_last_error.c_str(); }
int32_t fc_abi_version(void) { return FC_ABI_VERSION; }

}  // extern "C"
