// fc_jpeg.cpp -- the JPEG image front end of libfc.so (NEXT-4):
// "JPEG is decoded via dedicated hardware".  nvJPEG decodes
// a baseline 4:2:0 JPEG into caller-owned device I420 planes (Y, Cb, Cr); the
// planes are an FC_SURFACE_I420 surface, so the fused kernel turns them into
// tokens with the full-range BT.601 matrix (JFIF, FC_COLOR_BT601_FULL) like
// any decoded video frame.  The decoder itself is library code (the hardware
// JPEG engines through nvJPEG's hardware backend when this GPU and driver
// offer it, else nvJPEG's CUDA backend); parity starts at its output planes.
#include <nvjpeg.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "fc_internal.h"

struct fc_jpeg_decoder_s {
  nvjpegHandle_t handle = nullptr;
  nvjpegJpegState_t state = nullptr;
  int backend = 0;       // FC_JPEG_BACKEND_*
  bool batched = false;  // the hardware backend decodes through the batched API
  std::mutex mu;         // one decode at a time per decoder (nvJPEG state)
};

namespace fc {
namespace {

fc_status nvj_fail(nvjpegStatus_t s, const char* what) {
  const fc_status st = s == NVJPEG_STATUS_BAD_JPEG || s == NVJPEG_STATUS_INCOMPLETE_BITSTREAM
                           ? FC_ERR_INVALID_ARG
                       : s == NVJPEG_STATUS_JPEG_NOT_SUPPORTED || s == NVJPEG_STATUS_IMPLEMENTATION_NOT_SUPPORTED ||
                                 s == NVJPEG_STATUS_ARCH_MISMATCH  // e.g. no hardware backend for this GPU
                           ? FC_ERR_UNSUPPORTED
                       : s == NVJPEG_STATUS_ALLOCATOR_FAILURE ? FC_ERR_OOM
                                                              : FC_ERR_CUDA;
  return fail(st, std::string(what) + ": nvjpeg status " + std::to_string(static_cast<int>(s)));
}

// Destroys whatever part of a decoder exists.
void release(fc_jpeg_decoder_s* d) {
  if (d->state) nvjpegJpegStateDestroy(d->state);
  if (d->handle) nvjpegDestroy(d->handle);
  d->state = nullptr;
  d->handle = nullptr;
}

fc_status open_backend(fc_jpeg_decoder_s* d, int backend) {
  const nvjpegBackend_t b = backend == FC_JPEG_BACKEND_HARDWARE ? NVJPEG_BACKEND_HARDWARE : NVJPEG_BACKEND_DEFAULT;
  nvjpegStatus_t s = nvjpegCreateEx(b, nullptr, nullptr, 0, &d->handle);
  if (s != NVJPEG_STATUS_SUCCESS) {
    d->handle = nullptr;
    return nvj_fail(s, "nvjpegCreateEx");
  }
  s = nvjpegJpegStateCreate(d->handle, &d->state);
  if (s != NVJPEG_STATUS_SUCCESS) {
    release(d);
    return nvj_fail(s, "nvjpegJpegStateCreate");
  }
  d->batched = backend == FC_JPEG_BACKEND_HARDWARE;
  if (d->batched) {
    s = nvjpegDecodeBatchedInitialize(d->handle, d->state, 1, 1, NVJPEG_OUTPUT_YUV);
    if (s != NVJPEG_STATUS_SUCCESS) {
      release(d);
      return nvj_fail(s, "nvjpegDecodeBatchedInitialize");
    }
  }
  d->backend = backend;
  return FC_OK;
}

}  // namespace
}  // namespace fc

using namespace fc;

extern "C" {

fc_status fc_jpeg_decoder_create(int32_t backend, fc_jpeg_decoder_t** out) {
  if (!out) return fail(FC_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (backend != FC_JPEG_BACKEND_AUTO && backend != FC_JPEG_BACKEND_HARDWARE && backend != FC_JPEG_BACKEND_CUDA)
    return fail(FC_ERR_INVALID_ARG, "unknown JPEG backend");
  auto* d = new (std::nothrow) fc_jpeg_decoder_s();
  if (!d) return fail(FC_ERR_OOM, "decoder allocation");
  fc_status st = FC_ERR_UNSUPPORTED;
  if (backend != FC_JPEG_BACKEND_CUDA) st = open_backend(d, FC_JPEG_BACKEND_HARDWARE);
  if (st != FC_OK && backend != FC_JPEG_BACKEND_HARDWARE) st = open_backend(d, FC_JPEG_BACKEND_CUDA);
  if (st != FC_OK) {
    delete d;
    return st;
  }
  *out = d;
  return FC_OK;
}

void fc_jpeg_decoder_destroy(fc_jpeg_decoder_t* d) {
  if (!d) return;
  release(d);
  delete d;
}

int32_t fc_jpeg_decoder_backend(const fc_jpeg_decoder_t* d) { return d ? d->backend : -1; }

fc_status fc_jpeg_info(fc_jpeg_decoder_t* d, const uint8_t* data, size_t len, int32_t* width, int32_t* height,
                       int32_t* subsampling) {
  if (!d || !data || !len || !width || !height) return fail(FC_ERR_INVALID_ARG, "NULL argument");
  int nc = 0;
  nvjpegChromaSubsampling_t css;
  int w[NVJPEG_MAX_COMPONENT], h[NVJPEG_MAX_COMPONENT];
  const nvjpegStatus_t s = nvjpegGetImageInfo(d->handle, data, len, &nc, &css, w, h);
  if (s != NVJPEG_STATUS_SUCCESS) return nvj_fail(s, "nvjpegGetImageInfo");
  *width = w[0];
  *height = h[0];
  if (subsampling) *subsampling = nc == 3 && css == NVJPEG_CSS_420 ? FC_JPEG_420 : FC_JPEG_OTHER;
  return FC_OK;
}

fc_status fc_jpeg_decode_i420(fc_jpeg_decoder_t* d, const uint8_t* data, size_t len, const fc_nv12_surface* surf,
                              void* stream) {
  NvtxRange nvtx("fc_jpeg_decode_i420");
  if (!d || !data || !len || !surf || !surf->y || !surf->uv || !surf->v)
    return fail(FC_ERR_INVALID_ARG, "NULL argument");
  int32_t w = 0, h = 0, css = 0;
  fc_status st = fc_jpeg_info(d, data, len, &w, &h, &css);
  if (st != FC_OK) return st;
  if (css != FC_JPEG_420) return fail(FC_ERR_UNSUPPORTED, "only 3-component 4:2:0 JPEGs map onto I420 surfaces");
  if ((w & 1) || (h & 1)) return fail(FC_ERR_UNSUPPORTED, "odd image size (4:2:0 surfaces need even sizes)");
  if (surf->pitch_y < w || surf->pitch_uv < w / 2) return fail(FC_ERR_INVALID_ARG, "surface pitch too small");
  nvjpegImage_t img;
  std::memset(&img, 0, sizeof(img));
  img.channel[0] = const_cast<uint8_t*>(surf->y);
  img.channel[1] = const_cast<uint8_t*>(surf->uv);
  img.channel[2] = const_cast<uint8_t*>(surf->v);
  img.pitch[0] = static_cast<size_t>(surf->pitch_y);
  img.pitch[1] = img.pitch[2] = static_cast<size_t>(surf->pitch_uv);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  std::lock_guard<std::mutex> lk(d->mu);
  nvjpegStatus_t r;
  if (d->batched) {
    const unsigned char* const ptrs[1] = {data};
    const size_t lens[1] = {len};
    r = nvjpegDecodeBatched(d->handle, d->state, ptrs, lens, &img, s);
  } else {
    r = nvjpegDecode(d->handle, d->state, data, len, NVJPEG_OUTPUT_YUV, &img, s);
  }
  if (r != NVJPEG_STATUS_SUCCESS) return nvj_fail(r, d->batched ? "nvjpegDecodeBatched" : "nvjpegDecode");
  return FC_OK;
}

namespace {
struct MjpegJob {
  const uint8_t* const* data;
  const size_t* lengths;
  const fc_nv12_surface* surfaces;
  int64_t n;
  int32_t segments;
  std::vector<fc_jpeg_decoder_t*> dec;
  std::vector<cudaStream_t> streams;
  std::mutex mu;
  fc_status first = FC_OK;
  std::string first_msg;
};

// One GOP_s segment on worker w's decoder and stream: the targets
// [s*n/S, (s+1)*n/S), then a wait for the stream (the unit is busy until then).
int32_t mjpeg_segment(void* ctx, int64_t s, int32_t w) {
  auto* j = static_cast<MjpegJob*>(ctx);
  const int64_t b = s * j->n / j->segments, e = (s + 1) * j->n / j->segments;
  fc_status st = FC_OK;
  for (int64_t i = b; i < e && st == FC_OK; ++i)
    st = fc_jpeg_decode_i420(j->dec[w], j->data[i], j->lengths[i], &j->surfaces[i], j->streams[w]);
  if (st == FC_OK && cudaStreamSynchronize(j->streams[w]) != cudaSuccess) st = fail(FC_ERR_CUDA, "decode stream");
  if (st != FC_OK) {
    std::lock_guard<std::mutex> lk(j->mu);
    if (j->first == FC_OK) {
      j->first = st;
      j->first_msg = fc_last_error();
    }
    return static_cast<int32_t>(st);
  }
  return 0;
}
}  // namespace

fc_status fc_decode_mjpeg(const uint8_t* const* data, const size_t* lengths, int64_t n,
                          const fc_nv12_surface* surfaces, int32_t num_segments, int32_t num_workers,
                          int32_t max_in_flight, int32_t backend, int64_t* trace) {
  if (n < 0 || (n > 0 && (!data || !lengths || !surfaces)) || num_segments < 1 || num_workers < 1 ||
      max_in_flight < 1)
    return fail(FC_ERR_INVALID_ARG, "bad MJPEG decode arguments");
  if (n == 0) return FC_OK;
  MjpegJob j;
  j.data = data;
  j.lengths = lengths;
  j.surfaces = surfaces;
  j.n = n;
  j.segments = static_cast<int32_t>(std::min<int64_t>(num_segments, n));
  const int32_t workers = std::min(num_workers, j.segments);
  fc_status st = FC_OK;
  for (int w = 0; w < workers && st == FC_OK; ++w) {
    fc_jpeg_decoder_t* d = nullptr;
    st = fc_jpeg_decoder_create(backend, &d);
    if (st != FC_OK) break;
    j.dec.push_back(d);
    cudaStream_t s = nullptr;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) {
      st = fail(FC_ERR_CUDA, "decode stream");
      break;
    }
    j.streams.push_back(s);
  }
  if (st == FC_OK) {
    std::vector<int32_t> worker_of(j.segments);
    for (int32_t s = 0; s < j.segments; ++s) worker_of[s] = s % workers;  // round-robin GOP_s_VEC per worker
    st = fc_dispatch_segments(worker_of.data(), j.segments, workers, max_in_flight, mjpeg_segment, &j, trace);
    if (st != FC_OK && j.first != FC_OK) st = fail(j.first, j.first_msg);
  }
  for (cudaStream_t s : j.streams) cudaStreamDestroy(s);
  for (fc_jpeg_decoder_t* d : j.dec) fc_jpeg_decoder_destroy(d);
  return st;
}

}  // extern "C"
