/*
 * fc_oracle.c -- the CPU ORACLE for the FlashCodec preprocessing hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product (paper_2512_17574_b200/) never links, imports or executes it,
 * and shares no code, header, table or constant generator with it.
 *
 * It is the plain, slow, single-device definition of what the path computes
 * ("the compression outputs must remain consistent with those
 * produced on a single GPU"), written scalar and in the order the definitions
 * state.  Compile with -O2 -ffp-contract=off so that every double/float
 * operation rounds exactly as written (no FMA contraction).
 *
 * Functions and what pins them (tests/test_oracle_pins.py):
 *   oracle_nv12_to_rgb      O7  integer BT.601 limited range.
 *                               Pinned: exhaustive 2^24 closed-form check
 *                               against float BT.601 (<=1 LSB) + colour bars.
 *   oracle_yuv_pixel        R15 variants (BT.709, full range; NEXT-4).
 *                               Pinned: exhaustive 2^24 vs the float matrix
 *                               from (Kr, Kb) (<=2 LSB), black/white/grey
 *                               points, matrix 0 == oracle_bt601_pixel.
 *   oracle_resize_bicubic   O8  Pillow 12 ImagingResample BICUBIC, 8bpc path
 *                               (SURVEY D4).  Pinned: bit-exact vs
 *                               PIL.Image.resize on many shapes.
 *   oracle_normalize        O9  HF rescale (f64 multiply -> f32) then f32
 *                               (x-mean)/std.  Pinned: vs HF
 *                               numpy functions, all 768 values.
 *   oracle_tokens           O10-O11 pad with last frame + Qwen2-VL
 *                               patch order.  Pinned: vs HF
 *                               Qwen2VLVideoProcessor layout, brute-force
 *                               index encoding.
 *   oracle_preprocess       O7..O11 end to end.  Pinned: vs HF
 *                               Qwen2VLImageProcessorPil on oracle RGB.
 *   backend = 1 (R21)       torch's uint8 antialiased bicubic (precision
 *                               rule in make_coeffs) + HF's fused
 *                               normalisation.  Pinned: bit-exact vs torch
 *                               interpolate(antialias=True) on 8 shapes, HF
 *                               rescale_and_normalize (768 values) and HF
 *                               Qwen2VLVideoProcessor end to end.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ O7 -- */
/* C=Y-16, D=U-128, E=V-128;
 *   R = clamp((298C + 409E + 128) >> 8), G = clamp((298C - 100D - 208E + 128) >> 8),
 *   B = clamp((298C + 516D + 128) >> 8); >> is an arithmetic (floor) shift.
 * NV12: UV plane interleaved U,V at uv[(y/2)*pitch + 2*(x/2) + {0,1}]. */
static int clamp255(int v) { return v < 0 ? 0 : (v > 255 ? 255 : v); }

static int floor_div256(int v) {
  /* arithmetic shift == floor division by 256, written without relying on
   * implementation-defined >> of negatives */
  int q = v / 256;
  if ((v % 256) != 0 && v < 0) q -= 1;
  return q;
}

void oracle_bt601_pixel(int Y, int U, int V, uint8_t* rgb) {
  int C = Y - 16, D = U - 128, E = V - 128;
  rgb[0] = (uint8_t)clamp255(floor_div256(298 * C + 409 * E + 128));
  rgb[1] = (uint8_t)clamp255(floor_div256(298 * C - 100 * D - 208 * E + 128));
  rgb[2] = (uint8_t)clamp255(floor_div256(298 * C + 516 * D + 128));
}

/* Reading R15 (SURVEY 8(f) NEXT-4 variants; the paper is silent): the same
 * 8-bit fixed-point form for other matrices.  From the standard's luma
 * weights (Kr, Kb), Kg = 1-Kr-Kb, and the range (limited: Y scale 255/219,
 * chroma scale 255/224, Y offset 16; full: 1, 1, 0):
 *   R = Y + 2(1-Kr) E,  G = Y - 2(1-Kb)Kb/Kg D - 2(1-Kr)Kr/Kg E,  B = Y + 2(1-Kb) D,
 * every coefficient scaled by 256 and rounded to the nearest integer, then
 *   out = clamp((cY*(Y-y0) + cU*(U-128) + cV*(V-128) + 128) >> 8).
 * matrix: 0 BT.601 limited (== oracle_bt601_pixel), 1 BT.709 limited,
 * 2 BT.601 full, 3 BT.709 full. */
void oracle_yuv_coeffs(int matrix, int* k /* cY, y0, cRV, cGU, cGV, cBU */) {
  const double kr = (matrix == 1 || matrix == 3) ? 0.2126 : 0.299;
  const double kb = (matrix == 1 || matrix == 3) ? 0.0722 : 0.114;
  const double kg = 1.0 - kr - kb;
  const int limited = matrix <= 1;
  const double ys = limited ? 255.0 / 219.0 : 1.0;
  const double cs = limited ? 255.0 / 224.0 : 1.0;
  k[0] = (int)lround(256.0 * ys);
  k[1] = limited ? 16 : 0;
  k[2] = (int)lround(256.0 * 2.0 * (1.0 - kr) * cs);
  k[3] = (int)lround(-256.0 * 2.0 * (1.0 - kb) * kb / kg * cs);
  k[4] = (int)lround(-256.0 * 2.0 * (1.0 - kr) * kr / kg * cs);
  k[5] = (int)lround(256.0 * 2.0 * (1.0 - kb) * cs);
}

void oracle_yuv_pixel(int Y, int U, int V, int matrix, uint8_t* rgb) {
  int k[6];
  oracle_yuv_coeffs(matrix, k);
  int C = Y - k[1], D = U - 128, E = V - 128;
  rgb[0] = (uint8_t)clamp255(floor_div256(k[0] * C + k[2] * E + 128));
  rgb[1] = (uint8_t)clamp255(floor_div256(k[0] * C + k[3] * D + k[4] * E + 128));
  rgb[2] = (uint8_t)clamp255(floor_div256(k[0] * C + k[5] * D + 128));
}

/* every (Y, U, V) -> out[((Y*256 + U)*256 + V)*3 + c], for the exhaustive pins */
void oracle_yuv_table(int matrix, uint8_t* out) {
  for (int Y = 0; Y < 256; ++Y)
    for (int U = 0; U < 256; ++U)
      for (int V = 0; V < 256; ++V) oracle_yuv_pixel(Y, U, V, matrix, out + (((size_t)Y * 256 + U) * 256 + V) * 3);
}

void oracle_nv12_to_rgb_m(const uint8_t* y, int64_t pitch_y, const uint8_t* uv, int64_t pitch_uv,
                          int width, int height, int matrix, uint8_t* rgb /* height*width*3 */) {
  for (int r = 0; r < height; ++r)
    for (int c = 0; c < width; ++c) {
      int Y = y[(int64_t)r * pitch_y + c];
      int U = uv[(int64_t)(r / 2) * pitch_uv + 2 * (c / 2) + 0];
      int V = uv[(int64_t)(r / 2) * pitch_uv + 2 * (c / 2) + 1];
      if (matrix == 0) oracle_bt601_pixel(Y, U, V, rgb + ((int64_t)r * width + c) * 3);
      else oracle_yuv_pixel(Y, U, V, matrix, rgb + ((int64_t)r * width + c) * 3);
    }
}

void oracle_nv12_to_rgb(const uint8_t* y, int64_t pitch_y, const uint8_t* uv, int64_t pitch_uv,
                        int width, int height, uint8_t* rgb /* height*width*3 */) {
  oracle_nv12_to_rgb_m(y, pitch_y, uv, pitch_uv, width, height, 0, rgb);
}

/* ------------------------------------------------------------------ O8 -- */
/* Pillow ImagingResample, BICUBIC (a = -0.5, support 2), SURVEY O8:
 *   scale = in/out; fs = max(scale,1); support = 2*fs; ksize = 2*ceil(support)+1
 *   center = (o+0.5)*scale; xmin = max(0,(int)(center-support+0.5));
 *   xmax = min(in,(int)(center+support+0.5)); w_k = cubic((xmin+k-center+0.5)/fs)
 *   normalise by the sequential sum; iw = (int)(w<0 ? w*2^22-0.5 : w*2^22+0.5)
 *   out = clip8(2^21 + sum_k px*iw), clip8(v) = v>=2^30 ? 255 : v<=0 ? 0 : v>>22 */
static double cubic(double x) {
  const double a = -0.5;
  if (x < 0.0) x = -x;
  if (x < 1.0) return ((a + 2.0) * x - (a + 3.0)) * x * x + 1;
  if (x < 2.0) return (((x - 5) * x + 8) * x - 4) * a;
  return 0.0;
}

#define PRECISION_BITS 22

/* Backends (reading R21): 0 = HF's PIL-backend processor (Pillow,
 * PRECISION_BITS = 22); 1 = HF's torchvision-backend processor on CPU, whose
 * uint8 antialiased bicubic (torch.nn.functional.interpolate(antialias=True)
 * on uint8, ATen's Pillow port) uses the same windows and double weights but
 * rounds them at a precision p chosen per axis: the largest p < 22 with
 * (int)(0.5 + wmax * 2^(p+1)) < 2^15, wmax the largest normalised weight of
 * the axis (int16 weights); each pass is clamp((2^(p-1) + sum px*iw) >> p).
 * Pinned bit-exact against torch (tests/test_oracle_pins.py). */
typedef struct {
  int ksize;
  int prec;   /* fixed-point bits of iw */
  int* xmin;  /* [out] */
  int* cnt;   /* [out] */
  int* iw;    /* [out*ksize] */
} coeffs_t;

static int make_coeffs(int in, int out, int backend, coeffs_t* c) {
  double scale = (double)in / (double)out;
  double filterscale = scale < 1.0 ? 1.0 : scale;
  double support = 2.0 * filterscale;
  int ksize = (int)ceil(support) * 2 + 1;
  double* k = (double*)calloc((size_t)out * ksize, sizeof(double)); /* normalised weights, all outputs */
  c->ksize = ksize;
  c->xmin = (int*)malloc(sizeof(int) * out);
  c->cnt = (int*)malloc(sizeof(int) * out);
  c->iw = (int*)calloc((size_t)out * ksize, sizeof(int));
  if (!k || !c->xmin || !c->cnt || !c->iw) return -1;
  double wmax = 0.0;
  for (int o = 0; o < out; ++o) {
    double center = (o + 0.5) * scale;
    double ww = 0.0;
    double ss = 1.0 / filterscale;
    int xmin = (int)(center - support + 0.5);
    if (xmin < 0) xmin = 0;
    int xmax = (int)(center + support + 0.5);
    if (xmax > in) xmax = in;
    xmax -= xmin;
    double* kk = k + (size_t)o * ksize;
    for (int x = 0; x < xmax; ++x) {
      double w = cubic((x + xmin - center + 0.5) * ss);
      kk[x] = w;
      ww += w;
    }
    for (int x = 0; x < xmax; ++x)
      if (ww != 0.0) kk[x] /= ww;
    for (int x = 0; x < xmax; ++x)
      if (kk[x] > wmax) wmax = kk[x];
    c->xmin[o] = xmin;
    c->cnt[o] = xmax;
  }
  int prec = PRECISION_BITS;
  if (backend == 1)
    for (prec = 0; prec < 22; ++prec)
      if ((int)(0.5 + wmax * (1 << (prec + 1))) >= (1 << 15)) break;
  c->prec = prec;
  for (int o = 0; o < out; ++o)
    for (int x = 0; x < c->cnt[o]; ++x) {
      double w = k[(size_t)o * ksize + x];
      c->iw[(size_t)o * ksize + x] = (int)(w < 0 ? -0.5 + w * (1 << prec) : 0.5 + w * (1 << prec));
    }
  free(k);
  return 0;
}

static void free_coeffs(coeffs_t* c) {
  free(c->xmin);
  free(c->cnt);
  free(c->iw);
}

static uint8_t clip8(int64_t v, int prec) {
  if (v >= ((int64_t)1 << prec << 8)) return 255;
  if (v <= 0) return 0;
  return (uint8_t)(v >> prec);
}

/* Exposed for tests: the integer coefficient table of one axis (its
 * precision in *prec when prec != NULL). */
int oracle_resize_coeffs(int in, int out, int backend, int* xmin, int* cnt, int* iw, int ksize_cap, int* prec) {
  coeffs_t c;
  if (make_coeffs(in, out, backend, &c) != 0) return -1;
  if (prec) *prec = c.prec;
  int ks = c.ksize;
  if (ks <= ksize_cap) {
    memcpy(xmin, c.xmin, sizeof(int) * out);
    memcpy(cnt, c.cnt, sizeof(int) * out);
    memcpy(iw, c.iw, sizeof(int) * (size_t)out * ks);
  }
  free_coeffs(&c);
  return ks;
}

/* Pillow order (both backends): horizontal pass (all rows, u8 result) then
 * vertical pass. */
int oracle_resize_bicubic(const uint8_t* in, int w, int h, int w2, int h2, int backend, uint8_t* out) {
  const uint8_t* src = in;
  uint8_t* tmp = NULL;
  int cw = w;
  if (w2 != w) {
    coeffs_t c;
    if (make_coeffs(w, w2, backend, &c) != 0) return -1;
    tmp = (uint8_t*)malloc((size_t)h * w2 * 3);
    if (!tmp) return -1;
    for (int y = 0; y < h; ++y)
      for (int o = 0; o < w2; ++o)
        for (int ch = 0; ch < 3; ++ch) {
          int64_t ss = (int64_t)1 << (c.prec - 1);
          for (int k = 0; k < c.cnt[o]; ++k)
            ss += (int64_t)src[((size_t)y * w + c.xmin[o] + k) * 3 + ch] * c.iw[(size_t)o * c.ksize + k];
          tmp[((size_t)y * w2 + o) * 3 + ch] = clip8(ss, c.prec);
        }
    free_coeffs(&c);
    src = tmp;
    cw = w2;
  }
  if (h2 != h) {
    coeffs_t c;
    if (make_coeffs(h, h2, backend, &c) != 0) return -1;
    for (int o = 0; o < h2; ++o)
      for (int x = 0; x < cw; ++x)
        for (int ch = 0; ch < 3; ++ch) {
          int64_t ss = (int64_t)1 << (c.prec - 1);
          for (int k = 0; k < c.cnt[o]; ++k)
            ss += (int64_t)src[((size_t)(c.xmin[o] + k) * cw + x) * 3 + ch] * c.iw[(size_t)o * c.ksize + k];
          out[((size_t)o * cw + x) * 3 + ch] = clip8(ss, c.prec);
        }
    free_coeffs(&c);
  } else {
    memcpy(out, src, (size_t)h * cw * 3);
  }
  free(tmp);
  return 0;
}

/* ------------------------------------------------------------------ O9 -- */
/* Backend 0 (PIL): HF rescale (float)((double)v * rescale_factor), then
 * normalize (x - mean)/std in float32 (transformers image_transforms.rescale
 * / normalize).  Backend 1 (torchvision, R21): HF fuses the two
 * (image_processing_backends.py _fuse_mean_std_and_rescale_factor): mean' =
 * f32(mean) * f32(1/rescale_factor), std' likewise, in float32; then
 * tvF.normalize: (f32(v) - mean') / std' in float32. */
float oracle_normalize(int v, int ch, const float* mean, const float* std, double rescale, int backend) {
  if (backend == 1) {
    float inv = (float)(1.0 / rescale);
    float m2 = mean[ch] * inv;
    float s2 = std[ch] * inv;
    float d = (float)v - m2;
    return d / s2;
  }
  float x = (float)((double)v * rescale);
  float d = x - mean[ch];
  return d / std[ch];
}

/* ------------------------------------------------------------- O10-O11 -- */
/* rows (t, hb, wb, hm, wm) x cols (c, tp, ph, pw); frame index 2t+tp, padded
 * with the last frame.  `rs` holds n resized frames h2 x w2 x 3. */
void oracle_tokens(const uint8_t* rs, int64_t n, int w2, int h2, const float* mean, const float* std,
                   double rescale, int backend, float* tokens) {
  const int P = 14, M = 2, TP = 2;
  int64_t gt = (n + TP - 1) / TP;
  int gh = h2 / P, gw = w2 / P;
  int64_t row = 0;
  for (int64_t t = 0; t < gt; ++t)
    for (int hb = 0; hb < gh / M; ++hb)
      for (int wb = 0; wb < gw / M; ++wb)
        for (int hm = 0; hm < M; ++hm)
          for (int wm = 0; wm < M; ++wm) {
            int64_t col = 0;
            for (int c = 0; c < 3; ++c)
              for (int tp = 0; tp < TP; ++tp)
                for (int ph = 0; ph < P; ++ph)
                  for (int pw = 0; pw < P; ++pw) {
                    int64_t f = TP * t + tp;
                    if (f > n - 1) f = n - 1; /* pad with the last frame */
                    int y = (hb * M + hm) * P + ph;
                    int x = (wb * M + wm) * P + pw;
                    int v = rs[(((size_t)f * h2 + y) * w2 + x) * 3 + c];
                    tokens[row * 1176 + col] = oracle_normalize(v, c, mean, std, rescale, backend);
                    ++col;
                  }
            ++row;
          }
}

/* NEXT-1 exchange format: the same R6 walk, storing the resized u8 value
 * itself (the "code") instead of its normalised token.  Pinned: normalising
 * the codes reproduces oracle_tokens exactly. */
void oracle_codes(const uint8_t* rs, int64_t n, int w2, int h2, uint8_t* codes) {
  const int P = 14, M = 2, TP = 2;
  int64_t gt = (n + TP - 1) / TP;
  int gh = h2 / P, gw = w2 / P;
  int64_t row = 0;
  for (int64_t t = 0; t < gt; ++t)
    for (int hb = 0; hb < gh / M; ++hb)
      for (int wb = 0; wb < gw / M; ++wb)
        for (int hm = 0; hm < M; ++hm)
          for (int wm = 0; wm < M; ++wm) {
            int64_t col = 0;
            for (int c = 0; c < 3; ++c)
              for (int tp = 0; tp < TP; ++tp)
                for (int ph = 0; ph < P; ++ph)
                  for (int pw = 0; pw < P; ++pw) {
                    int64_t f = TP * t + tp;
                    if (f > n - 1) f = n - 1;
                    int y = (hb * M + hm) * P + ph;
                    int x = (wb * M + wm) * P + pw;
                    codes[row * 1176 + col] = rs[(((size_t)f * h2 + y) * w2 + x) * 3 + c];
                    ++col;
                  }
            ++row;
          }
}

/* ------------------------------------------------------- end to end -- */
typedef struct {
  const uint8_t* const* y;
  const uint8_t* const* uv;
  const int64_t* pitch_y;
  const int64_t* pitch_uv;
  int64_t n;
  int w, h, w2, h2;
  uint8_t* rgb_src; /* optional n*h*w*3 */
  uint8_t* rgb_rs;  /* n*h2*w2*3 */
  int nthreads, tid;
  int matrix;
  int backend;
  int status;
} job_t;

static void* frame_worker(void* arg) {
  job_t* j = (job_t*)arg;
  uint8_t* src = (uint8_t*)malloc((size_t)j->h * j->w * 3);
  if (!src) { j->status = -1; return NULL; }
  for (int64_t f = j->tid; f < j->n; f += j->nthreads) {
    oracle_nv12_to_rgb_m(j->y[f], j->pitch_y[f], j->uv[f], j->pitch_uv[f], j->w, j->h, j->matrix, src);
    if (j->rgb_src) memcpy(j->rgb_src + (size_t)f * j->h * j->w * 3, src, (size_t)j->h * j->w * 3);
    if (oracle_resize_bicubic(src, j->w, j->h, j->w2, j->h2, j->backend, j->rgb_rs + (size_t)f * j->h2 * j->w2 * 3) != 0)
      j->status = -1;
  }
  free(src);
  return NULL;
}

/* The sampled frames (already selected, in order) -> tokens [ceil(n/2)*gh*gw, 1176]. */
int oracle_preprocess(const uint8_t* const* y, const uint8_t* const* uv, const int64_t* pitch_y,
                      const int64_t* pitch_uv, int64_t n, int w, int h, int w2, int h2,
                      const float* mean, const float* std, double rescale, float* tokens,
                      uint8_t* rgb_src, uint8_t* rgb_rs, int nthreads, int matrix, int backend) {
  if (n <= 0 || w2 % 28 || h2 % 28) return -1;
  if (nthreads < 1) nthreads = 1;
  uint8_t* rs = rgb_rs ? rgb_rs : (uint8_t*)malloc((size_t)n * h2 * w2 * 3);
  if (!rs) return -1;
  job_t* jobs = (job_t*)calloc(nthreads, sizeof(job_t));
  pthread_t* th = (pthread_t*)calloc(nthreads, sizeof(pthread_t));
  int status = 0;
  for (int i = 0; i < nthreads; ++i) {
    job_t j = {y, uv, pitch_y, pitch_uv, n, w, h, w2, h2, rgb_src, rs, nthreads, i, matrix, backend, 0};
    jobs[i] = j;
    if (nthreads == 1) frame_worker(&jobs[i]);
    else pthread_create(&th[i], NULL, frame_worker, &jobs[i]);
  }
  for (int i = 0; i < nthreads; ++i) {
    if (nthreads > 1) pthread_join(th[i], NULL);
    if (jobs[i].status) status = -1;
  }
  if (status == 0 && tokens) oracle_tokens(rs, n, w2, h2, mean, std, rescale, backend, tokens);
  free(jobs);
  free(th);
  if (!rgb_rs) free(rs);
  return status;
}
