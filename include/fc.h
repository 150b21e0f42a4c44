/*
 * fc.h -- C ABI of the B200-native FlashCodec preprocessing hot path.
 *
 * The library (paper_2512_17574_b200/libfc.so) turns the sampled, decoded
 * NV12 frames of one video request into Qwen2-VL patch tokens + grid_thw,
 * with the request's GOPs partitioned over W GPUs (one process per GPU) and
 * the token shards gathered to the encoder GPU.
 *
 * Citations: P:n = arXiv 2512.17574 line n; S:n = SPEC.md line n;
 * readings R1..R12 are listed in DESIGN.md ("Readings of the paper").
 *
 * The calls follow the paper's FlashCodec API shape:
 *   analyse_bitstream       ~ fc_plan        (metadata -> per-rank GOP plan)
 *   add_decoding_request +
 *   get_decoding_output     ~ fc_preprocess  (stream-async; result ready when
 *                                             the caller synchronises the stream)
 * and its deferred allocation rule: the caller allocates the token
 * buffer only after planning, from the sizes fc_plan_rank reports.
 *
 * Conventions for every entry point:
 *   - Status codes only; nothing throws across the ABI.  On error nothing has
 *     been enqueued and no output has been written ("report, do not guess",
 *     S:34; no partial effects).  fc_last_error() returns a
 *     thread-local message describing the last failure on the calling thread.
 *   - "device pointer" = memory of the CUDA device current on the calling
 *     thread; "host pointer" = ordinary CPU memory.
 *   - The library never frees caller memory.  Device buffers are borrowed
 *     until the enqueued stream work completes.
 *   - There is no CPU fallback: on a machine without a usable sm_100 device
 *     fc_preprocess returns FC_ERR_CUDA.
 */
#ifndef FC_H_
#define FC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FC_ABI_VERSION 6  /* 2: token_dtype + color in fc_model_cfg; tokens as void*
                             3: surface_format in fc_model_cfg, v plane in the surface
                             4: fc_exchange_schedule, fc_last_kernel, fc_assign_requests, fc_submit, fc_ipc_*
                             5: the paged buffer's page table (fc_pages_*), fc_paged_copy, FC_ERR_OUT_OF_PAGES
                             6: fc_model_cfg.backend: HF PIL or torchvision processor arithmetic */
#define FC_TOKEN_COLS 1176 /* 3 channels * 2 (temporal patch) * 14 * 14 */

typedef enum {
  FC_OK = 0,
  FC_ERR_INVALID_ARG = 1,     /* NULL / out-of-range argument, malformed meta */
  FC_ERR_EMPTY_SELECTION = 2, /* sampling yields n == 0 or n > N (HF ValueError) */
  FC_ERR_ASPECT_RATIO = 3,    /* max(H,W)/min(H,W) > 200 (smart_resize precondition) */
  FC_ERR_UNSUPPORTED = 4,     /* odd dims, pitch % 16, unaligned surface, filter too wide */
  FC_ERR_MISSING_SURFACE = 5, /* a surface this rank must read is NULL */
  FC_ERR_RANK = 6,            /* rank outside [0, world_size) */
  FC_ERR_OOM = 7,             /* host or device allocation failed */
  FC_ERR_CUDA = 8,            /* CUDA launch/config error, or no sm_100 device */
  FC_ERR_NCCL = 9,            /* NCCL call failed */
  FC_ERR_OUT_OF_PAGES = 10    /* paged buffer: free list too short (back-pressure) */
} fc_status;

/* Exact rational frame rate (e.g. 30000/1001). */
typedef struct {
  int64_t num, den;
} fc_rational;

/* Video metadata M (Alg. 1 l.2; SPEC VideoMeta S:17-23).
 * Frames are in presentation order, constant frame rate (reading R11).
 * GOP g = frames [gop_start[g], gop_start[g+1]) (last GOP ends at num_frames);
 * gop_start[0] == 0, strictly increasing, all < num_frames. */
typedef struct {
  int32_t width, height; /* luma size; both even and >= 2 */
  int64_t num_frames;    /* N >= 1 */
  fc_rational fps;       /* source frame rate, num > 0, den > 0 */
  int64_t num_gops;      /* >= 1 */
  const int64_t* gop_start; /* host pointer, num_gops entries; copied by fc_plan */
} fc_video_meta;

/* Frame-set policy for I.  R1: FPS_STRIDE = HF Qwen2VLVideoProcessor
 * sample_frames (idx_i = floor(i*N/n)); LINSPACE = round(i*(N-1)/(n-1));
 * EXPLICIT = caller-given strictly increasing list (odd counts are padded). */
typedef enum { FC_SAMPLE_FPS_STRIDE = 0, FC_SAMPLE_LINSPACE = 1, FC_SAMPLE_EXPLICIT = 2 } fc_sampling;

/* Token element type.  F32 is the HF processor's output
 * (the default, and what every BASELINE config measures).  BF16 is the fp32
 * token rounded to nearest-even bfloat16 -- exactly torch's
 * `.to(torch.bfloat16)` of the F32 result -- for encoders that consume bf16;
 * it halves the token bytes written (reading R16). */
typedef enum {
  FC_TOKENS_F32 = 0,
  FC_TOKENS_BF16 = 1,
  /* u8 "codes" (NEXT-1 exchange format): the resized RGB value (R4's clip8
   * result) of every token element, same [rows][1176] layout, 1 byte each.
   * fc_expand_tokens turns codes into F32/BF16 tokens (R5's table), so a
   * multi-GPU request can gather 1176-byte rows instead of 4704-byte ones. */
  FC_TOKENS_U8 = 2
} fc_token_dtype;

/* YUV -> RGB matrix (reading R3 for the default; R15 for the variants):
 * 8-bit fixed point, out = clamp((cY*(Y - y0) + cU*(U-128) + cV*(V-128) + 128) >> 8)
 * with the coefficients round(256 * the standard matrix entry), the limited
 * ("TV", Y in [16,235]) or full ("PC", JPEG) range, nearest 2x2 chroma. */
typedef enum {
  FC_COLOR_BT601_LIMITED = 0, /* 298, 409 / -100, -208 / 516 (default, R3) */
  FC_COLOR_BT709_LIMITED = 1, /* 298, 459 / -55, -136 / 541 */
  FC_COLOR_BT601_FULL = 2,    /* 256, 359 / -88, -183 / 454 */
  FC_COLOR_BT709_FULL = 3     /* 256, 403 / -48, -120 / 475 */
} fc_color;

/* Decoded-surface layout (north star: "decoded NV12/YUV420 GOP surfaces").
 * Both are 8-bit 4:2:0 with nearest 2x2 chroma; they differ only in where the
 * chroma bytes live, so both give the same RGB (R3/R15) for the same samples. */
typedef enum {
  FC_SURFACE_NV12 = 0, /* Y plane + one interleaved U,V plane (NVDEC's output, default) */
  FC_SURFACE_I420 = 1  /* Y plane + separate U and V planes (planar YUV420, "I420") */
} fc_surface_format;

/* Which HF processor backend's arithmetic the resize (a6, a7) and normalise
 * (a8) steps reproduce (reading R21; "selectable interpolation
 * algorithms").  Sampling, smart_resize, colour and patch layout are shared.
 *   FC_BACKEND_PIL: HF's PIL-backend processor -- Pillow Image.resize(BICUBIC)
 *     (22-bit fixed point, R4), then f32(f64(v)/255) and (x - mean)/std (R5).
 *   FC_BACKEND_TORCHVISION: HF's torchvision-backend processor on CPU --
 *     torch's uint8 antialiased bicubic (the same Pillow windows and double
 *     weights, rounded at the precision p < 22 that keeps the largest weight of
 *     the axis an int16: the largest p with (int)(0.5 + wmax*2^(p+1)) < 2^15;
 *     each pass clamp((2^(p-1) + sum px*iw) >> p) with a u8 intermediate), then
 *     HF's fused normalisation (f32(v) - mean*f32(1/rescale)) / (std*f32(1/rescale))
 *     in float32.  (On CUDA tensors torchvision resizes in float, whose bits
 *     depend on the device; this mode is the CPU uint8 path, bit for bit.) */
typedef enum { FC_BACKEND_PIL = 0, FC_BACKEND_TORCHVISION = 1 } fc_backend;

/* Model / preprocessing configuration (Qwen2-VL video processor defaults,
 * filled by fc_model_cfg_default). */
typedef struct {
  int32_t patch_size;          /* 14 (only 14 supported) */
  int32_t temporal_patch_size; /* T = 2 (only 2 supported) */
  int32_t merge_size;          /* 2 (only 2 supported) */
  int64_t min_pixels;          /* 128*28*28 = 100352 (R2) */
  int64_t max_pixels;          /* 768*28*28 = 602112 (R2) */
  double total_pixels;         /* 0 = off; qwen-vl-utils total budget (R2 variant) */
  fc_sampling sampling;        /* FC_SAMPLE_FPS_STRIDE */
  double sample_fps;           /* 2.0 */
  int64_t num_frames;          /* 0 = use sample_fps; else HF num_frames rule */
  int32_t min_frames;          /* 4 */
  int32_t max_frames;          /* 768 */
  const int64_t* explicit_indices; /* host pointer, FC_SAMPLE_EXPLICIT only; copied */
  int64_t num_explicit;
  int32_t resized_height;      /* 0 = smart_resize; else fixed, multiple of 28 (224) */
  int32_t resized_width;
  float image_mean[3];         /* OpenAI CLIP mean */
  float image_std[3];          /* OpenAI CLIP std */
  double rescale_factor;       /* 1/255 */
  int32_t world_size;          /* W >= 1: GPUs the request is partitioned over */
  int32_t encoder_rank;        /* rank that receives the gathered tokens (default 0) */
  fc_token_dtype token_dtype;  /* FC_TOKENS_F32 (default) or FC_TOKENS_BF16 */
  fc_color color;              /* FC_COLOR_BT601_LIMITED (default) */
  fc_surface_format surface_format; /* FC_SURFACE_NV12 (default) or FC_SURFACE_I420 (ABI 3) */
  fc_backend backend;          /* FC_BACKEND_PIL (default) or FC_BACKEND_TORCHVISION (ABI 6) */
} fc_model_cfg;

void fc_model_cfg_default(fc_model_cfg* cfg);

/* Opaque, immutable plan.  Safe to share between threads; per-device
 * coefficient tables are created lazily inside it under a mutex.  Do not
 * destroy a plan while work that uses it is in flight. */
typedef struct fc_plan_s fc_plan_t;

/* fc_plan -- the planning half of Alg. 1 (l.1-4): frame sampling
 * (R1), smart_resize (R2), GOP->rank partition (get_GOPs_per_rank, R8) with
 * method-b temporal alignment (make_align_to_temporal_patch_size),
 * last-frame padding on the last rank, Pillow bicubic coefficient
 * tables (R4) and the normalisation table (R5).  Host only; no CUDA call.
 * *out receives a new plan (free with fc_plan_destroy) or NULL on error. */
fc_status fc_plan(const fc_video_meta* meta, const fc_model_cfg* cfg, fc_plan_t** out);
void fc_plan_destroy(fc_plan_t* plan);

typedef struct {
  int64_t grid_thw[3];      /* (ceil(n/2), H'/14, W'/14) */
  int32_t resized_h, resized_w;
  int64_t num_sampled;      /* n = |I| */
  int64_t pad_frames;       /* (-n) mod 2, applied on the last non-empty rank */
  int64_t token_rows;       /* grid_thw product */
  int64_t token_cols;       /* 1176 */
  double sampled_fps;       /* n / N * fps_src */
  double second_per_grid;   /* T / sampled_fps (Qwen2.5-VL metadata) */
  int32_t ranks_used;       /* non-empty ranks (empty ones are compacted to the end) */
  int32_t world_size;
  int32_t max_taps_h, max_taps_v; /* widest resize window per axis */
} fc_plan_info;

fc_status fc_plan_info_get(const fc_plan_t* plan, fc_plan_info* info);
/* Copies the n sampled frame indices (ascending) into host array `out`. */
fc_status fc_plan_sampled_indices(const fc_plan_t* plan, int64_t* out);

/* Rank r's share (Alg. 1 GOPs_VEC).  Owned GOPs [gop_begin,
 * gop_end); under method b a rank may additionally decode one frame of the
 * next GOP (tail_gop, tail_frame; -1 if none).  Its sampled frames are
 * sampled[sampled_begin .. sampled_begin+sampled_count) followed by pad_frames
 * copies of the last one; its token rows are [row_begin, row_end) of the
 * single-GPU result.  est_decode_frames = frames NVDEC would decode
 * (keyframe .. last target per GOP) -- reported, decode is out of scope. */
typedef struct {
  int64_t gop_begin, gop_end, tail_gop, tail_frame;
  int64_t sampled_begin, sampled_count, pad_frames;
  int64_t row_begin, row_end;
  int64_t est_decode_frames;
} fc_rank_plan;

fc_status fc_plan_rank(const fc_plan_t* plan, int32_t rank, fc_rank_plan* out);

/* fc_assign_requests -- throughput mode (many
 * independent requests, "replicas only"): place whole requests on GPUs by LPT
 * (longest processing time first) on their temporal-pair counts; no request
 * is split, so no exchange is needed (the per-request GOP split of P:339-340
 * is for latency mode).
 *   pairs:   host array [n], each request's temporal pairs (its work), >= 0
 *   rank_of: host array [n], written: the GPU of each request
 * Requests are taken in decreasing pairs (ties: lower index first), each to
 * the currently least-loaded rank (ties: lower rank); makespan <= 4/3 of the
 * optimum (Graham).  Host only.  n < 0, world < 1 or NULL arrays with n > 0 ->
 * FC_ERR_INVALID_ARG. */
fc_status fc_assign_requests(const int64_t* pairs, int32_t n, int32_t world, int32_t* rank_of);

/* One decoded frame in device memory (layout: the plan's cfg.surface_format).
 *   FC_SURFACE_NV12: luma plane y (height rows x pitch_y bytes) and the
 *     interleaved U,V plane uv (height/2 rows x pitch_uv bytes, >= width);
 *     v is ignored (NULL).
 *   FC_SURFACE_I420: luma plane y, U plane uv and V plane v (height/2 rows x
 *     pitch_uv bytes each, >= width/2; U and V share the pitch).
 * All plane pointers 16-byte aligned; pitches multiples of 16 and >= width
 * (y) / the chroma width above.  Surfaces must stay valid until the enqueued
 * work completes. */
typedef struct {
  const uint8_t* y;
  const uint8_t* uv;
  int64_t pitch_y, pitch_uv;
  const uint8_t* v;  /* ABI 3: V plane of an I420 surface, else NULL */
} fc_nv12_surface;
typedef fc_nv12_surface fc_yuv_surface;

/* fc_preprocess -- Alg. 1 l.21-22 (convert_AVframes_to_tensor_and_resize)
 * for rank `rank`: one fused kernel launch on `stream` computing, for the
 * rank's sampled frames, NV12 -> RGB (cfg.color; BT.601 limited by default,
 * R3) -> Pillow bicubic resize (R4) -> rescale + normalise (R5) -> temporal
 * pad + 14x14x2 patchify in 2x2 merge order (R6).
 *   surfaces:     host array of num_surfaces descriptors indexed by GLOBAL
 *                 frame index (0..N-1); entries this rank does not read may
 *                 have NULL pointers (FC_ERR_MISSING_SURFACE otherwise).
 *   tokens:       device pointer, (row_end-row_begin) x 1176 elements of
 *                 cfg.token_dtype (fp32 by default, or bf16), contiguous.
 *   grid_thw:     host out (3 values) or NULL.
 *   stream:       cudaStream_t (0 = legacy default stream).
 * Asynchronous: returns after enqueueing.  Validation happens before any
 * launch.  A rank with no rows returns FC_OK without launching. */
fc_status fc_preprocess(const fc_plan_t* plan, int32_t rank, const fc_nv12_surface* surfaces,
                        int64_t num_surfaces, void* tokens, int64_t grid_thw[3], void* stream);

/* fc_submit -- plan one request and enqueue its preprocessing in ONE call
 * (FlashCodec's add_decoding_request: analyse + submit): exactly
 * fc_plan(meta, cfg) followed by fc_preprocess(plan, rank, ...), for the
 * small-request path where per-call host overhead dominates (config 1: a
 * ~12 us kernel).  *plan_out receives the plan (caller-owned: fc_plan_destroy
 * after the stream work completes); on any error nothing is enqueued and
 * *plan_out is NULL.  tokens: (row_end-row_begin) x 1176 of cfg.token_dtype,
 * sized by the caller from the request's shape (fc_plan_rank of an equal
 * request, or the closed form of fc_plan_info). */
fc_status fc_submit(const fc_video_meta* meta, const fc_model_cfg* cfg, int32_t rank, const fc_nv12_surface* surfaces,
                    int64_t num_surfaces, void* tokens, void* stream, fc_plan_t** plan_out);

/* Same, additionally dumping the integer intermediates for parity tests:
 *   rgb_src:     device u8 [n_r, H, W, 3]  (BT.601 output) or NULL
 *   rgb_resized: device u8 [n_r, H', W', 3] (resize output)  or NULL
 * where n_r = the rank's frames including padding, in order. */
fc_status fc_preprocess_debug(const fc_plan_t* plan, int32_t rank, const fc_nv12_surface* surfaces,
                              int64_t num_surfaces, void* tokens, int64_t grid_thw[3], void* stream,
                              uint8_t* rgb_src, uint8_t* rgb_resized);

/* Throughput mode (config 5): `count` independent (plan, rank) jobs on
 * `stream`.  surfaces[i] / num_surfaces[i] / tokens[i] as in fc_preprocess
 * for job i (tokens[i] may be NULL for a job whose rank has no rows).  Every
 * job is validated before anything is launched.  Consecutive jobs with equal
 * source size, resized size and frame count form ONE persistent launch (the
 * work list spans all their pairs; per-job token bases and the NV12 tensor
 * maps travel in a small stream-ordered device descriptor), so a batch of
 * same-shape clips is a single kernel launch.  Jobs of other shapes start a
 * new launch.  Results equal per-job fc_preprocess calls bit for bit. */
fc_status fc_preprocess_batch(const fc_plan_t* const* plans, const int32_t* ranks, int32_t count,
                              const fc_nv12_surface* const* surfaces, const int64_t* num_surfaces,
                              void* const* tokens, void* stream);

/* NEXT-2 -- paged token output (Fig. 10; SPEC embed_buffer
 * write_chunk).  The rank's token rows are written, in order, as ONE write
 * chunk of a paged embedding buffer, straight from the kernel's epilogue (no
 * linear staging buffer): row i of the rank goes to pool row
 *     page_ids[s / page_rows] * page_rows + s % page_rows,   s = first_offset + i.
 *   pool:          device pointer, pool_pages pages of page_rows x 1176 tokens
 *                  (element type cfg.token_dtype: F32 or BF16).
 *   page_rows:     tokens per page; a power of two.
 *   page_ids:      HOST array of num_pages page ids -- the request's
 *                  pv_page_indices segment for this write -- each in
 *                  [0, pool_pages); copied (uploaded with the launch).
 *   first_offset:  pv_cu_page_len mod page_rows (tokens already in the first
 *                  page), in [0, page_rows).
 * num_pages must cover ceil((first_offset + rows) / page_rows).  Rows of other
 * requests in the same pages are untouched.  Errors as fc_preprocess, plus
 * FC_ERR_INVALID_ARG for an inconsistent page table (nothing is launched). */
typedef struct {
  void* pool;
  int64_t pool_pages;
  int32_t page_rows;
  int32_t num_pages;
  const int32_t* page_ids;
  int64_t first_offset;
} fc_paged_tokens;

fc_status fc_preprocess_paged(const fc_plan_t* plan, int32_t rank, const fc_nv12_surface* surfaces,
                              int64_t num_surfaces, const fc_paged_tokens* out, int64_t grid_thw[3], void* stream);

/* ---- NEXT-2: the paged embedding buffer (Fig. 10; SPEC
 * embed_buffer S:218-290) ----
 *
 * The buffer's page table is host bookkeeping (fc_pages_*); the data moves in
 * device kernels: fc_preprocess_paged (vision tokens straight from the pixel
 * kernel) and fc_paged_copy (read_chunk: pages -> a contiguous chunk, "materialise
 * into contiguous memory only at use time"; write_chunk: a contiguous
 * chunk -> pages).  Each iteration's reads or writes are described by the
 * paper's four indices (reading R21 in DESIGN.md):
 *   pv_indptr[i] .. pv_indptr[i+1]   request i's tokens in the iteration's
 *                                    contiguous chunk (CSR; count = difference)
 *   pv_page_indices[pv_page_indptr[i] .. pv_page_indptr[i+1]]
 *                                    the pages request i touches this iteration,
 *                                    in token order
 *   pv_cu_page_len[i]                tokens request i wrote (or read) in all
 *                                    previous iterations; its first token this
 *                                    iteration is token n = pv_cu_page_len[i] mod
 *                                    page_rows of the first listed page, and the
 *                                    next ones fill the listed pages in order. */
typedef struct {
  int32_t num_requests;
  const int64_t* pv_indptr;       /* [num_requests + 1], pv_indptr[0] == 0, non-decreasing */
  const int32_t* pv_page_indptr;  /* [num_requests + 1], pv_page_indptr[0] == 0, non-decreasing */
  const int32_t* pv_page_indices; /* [pv_page_indptr[num_requests]] page ids */
  const int64_t* pv_cu_page_len;  /* [num_requests], >= 0 */
} fc_ragged_index;

typedef enum { FC_PAGE_WRITE = 0, FC_PAGE_READ = 1 } fc_page_op;

/* The page table (SPEC PageTable): total_pages pages of page_rows
 * tokens (page_rows a power of two <= 2^20); a page is free or owned by
 * exactly one request; requests are caller-chosen int64 ids.  Not thread-safe
 * (one owner thread: the scheduler that builds the iteration).  Host only, no
 * CUDA call.  Errors: FC_ERR_INVALID_ARG, FC_ERR_OOM. */
typedef struct fc_pages_s fc_pages_t;
fc_status fc_pages_create(int64_t total_pages, int32_t page_rows, fc_pages_t** out);
void fc_pages_destroy(fc_pages_t* t);

/* alloc_pages: reserve room for `tokens` more tokens after what
 * request `req` has written (or had reserved) so far, appending the minimal
 * number of pages from the free list (lowest ids first); new_ids (may be NULL,
 * else capacity >= the pages appended) receives them, *n_new their count.
 * All or nothing: FC_ERR_OUT_OF_PAGES when the free list is too short (the
 * caller's back-pressure signal, nothing is allocated). */
fc_status fc_pages_alloc(fc_pages_t* t, int64_t req, int64_t tokens, int32_t* new_ids, int32_t capacity,
                         int32_t* n_new);

/* Build one iteration's ragged index for n requests: reqs[i] moves counts[i]
 * tokens (counts[i] >= 0; a request may appear once per call).
 *   FC_PAGE_WRITE: tokens go after the request's written ones; the pages must
 *     be allocated (FC_ERR_INVALID_ARG otherwise: SPEC CapacityError).
 *   FC_PAGE_READ: tokens follow the request's read ones, a prefix-ordered read
 *     of written tokens (FC_ERR_INVALID_ARG past the written count: SPEC
 *     UnwrittenRange).  Pages whose last token this read consumes become
 *     "consumed"; fc_pages_free_consumed releases them.
 * The cursors advance at this call (the caller orders the device work on a
 * stream).  Outputs are caller arrays: pv_indptr [n + 1], pv_page_indptr
 * [n + 1], pv_cu_page_len [n], pv_page_indices [capacity]; *num_indices = the
 * page ids written -- capacity too small -> FC_ERR_INVALID_ARG, *num_indices =
 * the size needed, nothing changes.  All or nothing on every error. */
fc_status fc_pages_index(fc_pages_t* t, fc_page_op op, const int64_t* reqs, const int64_t* counts, int32_t n,
                         int64_t* pv_indptr, int32_t* pv_page_indptr, int32_t* pv_page_indices, int32_t capacity,
                         int64_t* pv_cu_page_len, int32_t* num_indices);

/* Eager page free (Fig. 10: "processed blocks (e.g., 8 and 11) are
 * promptly freed"): return every consumed page to the free list; call it once
 * the iteration's read kernels have completed.  A page is consumed when a read
 * passes its last token, or when its request was released.  freed (may be
 * NULL) receives up to `capacity` ids in the order they were consumed;
 * *n_freed = how many were freed (all of them are, whatever the capacity). */
fc_status fc_pages_free_consumed(fc_pages_t* t, int32_t* freed, int32_t capacity, int32_t* n_freed);

/* A finished (or cancelled) request: all its pages become consumed (freed at
 * the next fc_pages_free_consumed) and its id is forgotten.  Unknown id ->
 * FC_ERR_INVALID_ARG. */
fc_status fc_pages_release(fc_pages_t* t, int64_t req);

/* Counters: free pages, pages owned by live requests, consumed pages awaiting
 * fc_pages_free_consumed, live requests (any pointer may be NULL).  free +
 * owned + consumed == total_pages always. */
fc_status fc_pages_stats(const fc_pages_t* t, int64_t* free_pages, int64_t* owned_pages, int64_t* consumed_pages,
                         int64_t* live_requests);

/* read_chunk / write_chunk on the device: moves the iteration's tokens between
 * the pool and a contiguous chunk, as `idx` says.
 *   op = FC_PAGE_READ:  chunk row pv_indptr[i] + k  <-  request i's k-th token
 *   op = FC_PAGE_WRITE: the same rows in the other direction
 * where request i's k-th token is pool row page * page_rows + s % page_rows,
 * page = pv_page_indices[pv_page_indptr[i] + s / page_rows], s = n + k,
 * n = pv_cu_page_len[i] mod page_rows.
 *   pool:      device pointer, pool_pages * page_rows rows of row_bytes
 *   chunk:     device pointer, pv_indptr[num_requests] rows of row_bytes
 *   row_bytes: a multiple of 8 (fp32 tokens 4704, bf16 2352, u8 codes 1176);
 *              pool and chunk 16-byte aligned.
 *   idx:       HOST arrays, validated (monotone pointers, enough pages for
 *              each request, ids inside the pool) and uploaded with the launch.
 * One HBM-bound kernel launch on `stream` (none for an empty chunk).  Errors:
 * FC_ERR_INVALID_ARG (nothing launched), FC_ERR_CUDA. */
fc_status fc_paged_copy(fc_page_op op, const fc_ragged_index* idx, void* pool, int64_t pool_pages, int32_t page_rows,
                        int64_t row_bytes, void* chunk, void* stream);

/* fc_expand_tokens -- R5 on u8 codes (FC_TOKENS_U8 output of fc_preprocess,
 * usually gathered from all ranks): tokens[r][i] = table[channel(i)][codes[r][i]]
 * with channel(i) = i / 392 (columns are (c, tp, ph, pw)).  The table is the
 * plan's normalisation (mean/std/rescale), in fp32 or rounded to bf16 (R16).
 *   codes:     device pointer, rows x 1176 u8, contiguous.
 *   tokens:    device pointer, rows x 1176 elements of out_dtype (F32 | BF16).
 * One HBM-bound kernel launch on `stream`; results equal fc_preprocess with
 * token_dtype = out_dtype bit for bit. */
fc_status fc_expand_tokens(const fc_plan_t* plan, int64_t rows, const uint8_t* codes, void* tokens,
                           fc_token_dtype out_dtype, void* stream);

/* ---- exchange: gather row shards to the encoder rank ---- */

/* NCCL communicator bootstrap without a torch type in the ABI: rank 0 calls
 * fc_nccl_unique_id (128 bytes into `id`), the caller broadcasts the bytes
 * over its process group, then every rank calls fc_nccl_comm_init with the
 * CUDA device already current.  Returned comm is an ncclComm_t. */
fc_status fc_nccl_unique_id(uint8_t id[128]);
fc_status fc_nccl_comm_init(const uint8_t id[128], int32_t world_size, int32_t rank, void** comm);
fc_status fc_nccl_comm_destroy(void* comm);

/* NEXT-1 -- column-split output ("the resulting patch token
 * embeddings are first generated, then split along the last dimension, and
 * finally each resulting chunk is written into the IPC patch buffer of the
 * corresponding GPU").  Same computation as fc_preprocess for rank `rank`, but
 * the rank's token rows are written as W = world_size column blocks straight
 * from the kernel's epilogue:
 *   blocks: device fp32 [W][rows_r][C], C = 1176 / W, rows_r = row_end - row_begin;
 *           block j holds columns [j*C, (j+1)*C) of the rank's rows, in row order.
 * Requires fp32 tokens, NV12 surfaces and W dividing 1176 (1..8 except 5);
 * FC_ERR_UNSUPPORTED otherwise.  Errors and asynchrony as fc_preprocess. */
fc_status fc_preprocess_colsplit(const fc_plan_t* plan, int32_t rank, const fc_nv12_surface* surfaces,
                                 int64_t num_surfaces, float* blocks, int64_t grid_thw[3], void* stream);

/* fc_scatter_columns -- the paper's "collective scatter" of the column
 * blocks: an all-to-all (grouped ncclSend/ncclRecv) after which rank j holds
 * columns [j*C, (j+1)*C) of ALL token rows:
 *   blocks: this rank's fc_preprocess_colsplit output (may be NULL if it has no rows)
 *   mine:   device fp32 [token_rows][C]; rank p's rows land at mine + row_begin_p*C
 *           (this rank's own block is copied in with cudaMemcpyAsync).
 * Collective: every rank of the plan's world must call it.  Async on stream. */
fc_status fc_scatter_columns(const fc_plan_t* plan, int32_t rank, void* comm, const float* blocks, float* mine,
                             void* stream);

/* fc_exchange_schedule -- the transfers one rank issues in an exchange step
 * (a10; reading R9): FC_XCHG_GATHER is what fc_gather runs (row
 * shards -> the encoder rank's full buffer), FC_XCHG_COLSPLIT what
 * fc_scatter_columns runs (column blocks, all-to-all).  Both functions execute
 * exactly this list, so it is the testable form of their offset arithmetic.
 *   src_offset: byte offset into the rank's send buffer (shard / blocks)
 *               for FC_XFER_SEND and FC_XFER_LOCAL;
 *   dst_offset: byte offset into its receive buffer (full / mine) for
 *               FC_XFER_RECV and FC_XFER_LOCAL;  bytes: length.
 * out may be NULL (then only *count is written); capacity too small ->
 * FC_ERR_INVALID_ARG with *count = the size needed.  Host only, no CUDA call. */
typedef enum { FC_XCHG_GATHER = 0, FC_XCHG_COLSPLIT = 1 } fc_exchange_kind;
typedef enum { FC_XFER_LOCAL = 0, FC_XFER_SEND = 1, FC_XFER_RECV = 2 } fc_xfer_dir;
typedef struct {
  int32_t peer;      /* the other rank (== rank for FC_XFER_LOCAL) */
  int32_t dir;       /* fc_xfer_dir */
  int64_t src_offset, dst_offset, bytes;
} fc_transfer;
fc_status fc_exchange_schedule(const fc_plan_t* plan, int32_t rank, fc_exchange_kind kind, fc_transfer* out,
                               int32_t capacity, int32_t* count);

/* CUDA IPC handles for the fused peer-store exchange (NEXT-1, P:527-530:
 * shards written straight into the encoder's IPC patch buffer).  The
 * encoder exports its token buffer once; every other rank imports it and
 * passes  peer_base + row_begin * row_bytes  as the `tokens` of fc_preprocess,
 * so its kernel's epilogue stores land in the encoder's HBM over NVLink while
 * the rank computes -- no separate gather pass.  The caller orders the
 * encoder's reads after every rank's kernel (e.g. a stream-ordered
 * collective or an interprocess event).
 *   fc_ipc_export: dev_ptr = the base of a cudaMalloc'd allocation (torch
 *                  tensors from the caching allocator: data_ptr() may be
 *                  inside a larger block -- export with its offset, see
 *                  fc_ipc_export_range); handle = 64 opaque bytes.
 *   fc_ipc_import: *dev_ptr = the allocation's base in this process (another
 *                  process; cudaIpcMemLazyEnablePeerAccess).
 *   fc_ipc_close:  releases an imported mapping.
 * Errors: FC_ERR_INVALID_ARG (NULL), FC_ERR_CUDA (the runtime's reason). */
fc_status fc_ipc_export(void* dev_ptr, uint8_t handle[64]);
/* the allocation containing ptr: its handle and ptr's byte offset in it */
fc_status fc_ipc_export_range(void* ptr, uint8_t handle[64], int64_t* offset);
fc_status fc_ipc_import(const uint8_t handle[64], void** dev_ptr);
fc_status fc_ipc_close(void* dev_ptr);

/* fc_gather -- gatherv of every rank's contiguous row shard into the encoder
 * rank's full token buffer (grouped ncclSend/ncclRecv, R9):
 *   shard: device pointer, this rank's (row_end-row_begin) x 1176 tokens
 *          (element type cfg.token_dtype)
 *   full:  encoder rank: device pointer token_rows x 1176 tokens (its own shard
 *          is copied in with cudaMemcpyAsync unless shard already aliases
 *          full + row_begin*1176); other ranks: ignored (may be NULL).
 * Collective: every rank of the plan's world must call it.  Async on stream. */
fc_status fc_gather(const fc_plan_t* plan, int32_t rank, void* comm, const void* shard, void* full,
                    void* stream);

/* ---- NEXT-4 images: "JPEG is decoded via dedicated hardware" ----
 * nvJPEG decodes one baseline, 3-component, 4:2:0 JPEG (JFIF YCbCr) into
 * caller-owned device planes laid out as an FC_SURFACE_I420 surface: Y in
 * surf->y (pitch_y), Cb in surf->uv and Cr in surf->v (pitch_uv).  Feed the
 * surface to fc_preprocess with cfg.surface_format = FC_SURFACE_I420 and
 * cfg.color = FC_COLOR_BT601_FULL (JFIF is full-range BT.601); a single image
 * is a one-frame request (num_frames 1, explicit index 0), padded to the
 * temporal patch like an odd frame count, grid (1, H'/14, W'/14).
 * The decoder is library code: the hardware JPEG engines (nvJPEG's hardware
 * backend) when the GPU and driver offer them, else nvJPEG's CUDA backend.
 * A decoder serialises its decodes (one nvJPEG state); use one per thread
 * for concurrency. */
typedef struct fc_jpeg_decoder_s fc_jpeg_decoder_t;
typedef enum {
  FC_JPEG_BACKEND_AUTO = 0,     /* hardware if available, else CUDA */
  FC_JPEG_BACKEND_HARDWARE = 1, /* the JPEG engines only (error if absent) */
  FC_JPEG_BACKEND_CUDA = 2      /* nvJPEG's CUDA decoder */
} fc_jpeg_backend;
typedef enum { FC_JPEG_420 = 0, FC_JPEG_OTHER = 1 } fc_jpeg_subsampling;
/* backend: fc_jpeg_backend.  Errors: FC_ERR_INVALID_ARG (NULL out, unknown
 * backend), FC_ERR_UNSUPPORTED / FC_ERR_CUDA (backend unavailable). */
fc_status fc_jpeg_decoder_create(int32_t backend, fc_jpeg_decoder_t** out);
void fc_jpeg_decoder_destroy(fc_jpeg_decoder_t* dec);
/* The backend a decoder opened (FC_JPEG_BACKEND_HARDWARE or _CUDA), -1 for NULL. */
int32_t fc_jpeg_decoder_backend(const fc_jpeg_decoder_t* dec);
/* Header parse on the host: luma size and whether the image is 3-component
 * 4:2:0 (FC_JPEG_420).  data: host pointer to the whole JPEG file, len bytes.
 * Errors: FC_ERR_INVALID_ARG (NULL, not a JPEG), FC_ERR_UNSUPPORTED. */
fc_status fc_jpeg_info(fc_jpeg_decoder_t* dec, const uint8_t* data, size_t len, int32_t* width, int32_t* height,
                       int32_t* subsampling);
/* Decode into `surf` (device planes, capacity >= height rows x pitch; the
 * caller keeps them alive) on `stream` (cudaStream_t; NULL = legacy default).
 * Requires a 4:2:0 image of even width and height (FC_ERR_UNSUPPORTED
 * otherwise) and pitch_y >= width, pitch_uv >= width/2 (FC_ERR_INVALID_ARG).
 * data is a host pointer; nothing is enqueued on error. */
fc_status fc_jpeg_decode_i420(fc_jpeg_decoder_t* dec, const uint8_t* data, size_t len, const fc_nv12_surface* surf,
                              void* stream);

/* ---- NEXT-3 (partial): stall-free GOP_s dispatch (Alg. 2) ----
 * A request's decode work is split into GOP_s segments (runs of GOPs a decode
 * unit decodes from their keyframe).  Worker w (of num_workers
 * threads, Alg. 2 l.6) runs its segments {s : worker_of[s] == w} in increasing
 * s by calling fn(ctx, s, w) on its own thread; at most max_in_flight
 * segments run at once (N decode units, l.10).  A worker that finishes a
 * segment and has more keeps its unit (l.12-13: "the remaining GOP_s within the
 * same worker is prioritized"); a worker that runs dry releases its
 * unit and wakes a waiting worker.  fn returns 0 on success; a nonzero return
 * stops new dispatches and the call returns FC_ERR_CUDA after the running
 * segments end.  trace (host, optional, 3 * num_segments int64): per
 * completion in order, (segment, worker, fn's return).  Blocks until every
 * segment has run.  Errors: FC_ERR_INVALID_ARG (negative counts, worker out
 * of range, NULL fn), FC_ERR_OOM. */
typedef int32_t (*fc_segment_fn)(void* ctx, int64_t segment, int32_t worker);
fc_status fc_dispatch_segments(const int32_t* worker_of, int64_t num_segments, int32_t num_workers,
                               int32_t max_in_flight, fc_segment_fn fn, void* ctx, int64_t* trace);

/* Decode the target frames of a Motion-JPEG request -- every frame an
 * independent 4:2:0 JPEG, i.e. a one-frame GOP, so only targets are decoded
 * -- into I420 surfaces through fc_dispatch_segments: the n targets
 * (data[i], lengths[i]: host pointers, in order) are cut into num_segments
 * contiguous GOP_s segments dealt round-robin to num_workers threads, each with
 * its own nvJPEG decoder (backend: fc_jpeg_backend) and CUDA stream; at most
 * max_in_flight segments decode at once.  surfaces[i] receives target i
 * (device planes as in fc_jpeg_decode_i420).  Returns after every decode has
 * completed on the device, so any stream may consume the surfaces.  trace as
 * in fc_dispatch_segments.  Errors: as fc_jpeg_decode_i420 (the first
 * failure), FC_ERR_INVALID_ARG for bad counts. */
fc_status fc_decode_mjpeg(const uint8_t* const* data, const size_t* lengths, int64_t n,
                          const fc_nv12_surface* surfaces, int32_t num_segments, int32_t num_workers,
                          int32_t max_in_flight, int32_t backend, int64_t* trace);

const char* fc_status_string(fc_status s);
const char* fc_last_error(void);
int32_t fc_abi_version(void);

/* Process-wide count of kernels this library has launched successfully
 * (fused preprocess kernels; NCCL's own kernels and memcpys not included).
 * Monotone; safe to call from any thread; no CUDA call. */
uint64_t fc_kernel_launches(void);

/* Which fused kernel the calling thread's last successful fc_preprocess*
 * launch used: FC_KERNEL_MMA (the mma.sync kernel, the default for every
 * request) or FC_KERNEL_TC (the tcgen05 kernel, selected with the environment
 * variable FC_TC=1 for NV12 surfaces, fp32 tokens and strip windows up to 255
 * source columns / 128 source rows per 16 output rows);
 * FC_KERNEL_NONE before any launch.  Thread-local, no CUDA call. */
typedef enum { FC_KERNEL_NONE = 0, FC_KERNEL_TC = 1, FC_KERNEL_MMA = 2 } fc_kernel_id;
int32_t fc_last_kernel(void);

#ifdef __cplusplus
}
#endif
#endif /* FC_H_ */
