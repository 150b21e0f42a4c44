"""ctypes declaration of the C ABI in include/fc.h (argument marshalling only).

Loading fails loudly when libfc.so is missing: there is no CPU or Python
fallback for any step of the path.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# FC_LIB_VARIANT (kernel A/B experiments only): load libfc_<variant>.so, a
# build of the same sources with a change under test, from this directory
LIB_PATH = os.path.join(HERE, f"libfc_{os.environ['FC_LIB_VARIANT']}.so" if os.environ.get("FC_LIB_VARIANT")
                        else "libfc.so")

FC_TOKEN_COLS = 1176
ABI_VERSION = 6  # include/fc.h FC_ABI_VERSION this binding marshals for
STATUS = {0: "FC_OK", 1: "FC_ERR_INVALID_ARG", 2: "FC_ERR_EMPTY_SELECTION", 3: "FC_ERR_ASPECT_RATIO",
          4: "FC_ERR_UNSUPPORTED", 5: "FC_ERR_MISSING_SURFACE", 6: "FC_ERR_RANK", 7: "FC_ERR_OOM",
          8: "FC_ERR_CUDA", 9: "FC_ERR_NCCL", 10: "FC_ERR_OUT_OF_PAGES"}
SAMPLING = {"fps_stride": 0, "linspace": 1, "explicit": 2}
TOKEN_DTYPES = {"f32": 0, "bf16": 1, "u8": 2}
COLORS = {"bt601": 0, "bt709": 1, "bt601_full": 2, "bt709_full": 3}
SURFACES = {"nv12": 0, "i420": 1}
BACKENDS = {"pil": 0, "torchvision": 1}


class FcError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        self.status = status
        self.name = STATUS.get(status, str(status))
        super().__init__(f"{where}: {self.name}: {detail}")


class Rational(ctypes.Structure):
    _fields_ = [("num", ctypes.c_int64), ("den", ctypes.c_int64)]


class VideoMetaC(ctypes.Structure):
    _fields_ = [("width", ctypes.c_int32), ("height", ctypes.c_int32), ("num_frames", ctypes.c_int64),
                ("fps", Rational), ("num_gops", ctypes.c_int64), ("gop_start", ctypes.POINTER(ctypes.c_int64))]


class ModelCfgC(ctypes.Structure):
    _fields_ = [("patch_size", ctypes.c_int32), ("temporal_patch_size", ctypes.c_int32),
                ("merge_size", ctypes.c_int32), ("min_pixels", ctypes.c_int64), ("max_pixels", ctypes.c_int64),
                ("total_pixels", ctypes.c_double), ("sampling", ctypes.c_int), ("sample_fps", ctypes.c_double),
                ("num_frames", ctypes.c_int64), ("min_frames", ctypes.c_int32), ("max_frames", ctypes.c_int32),
                ("explicit_indices", ctypes.POINTER(ctypes.c_int64)), ("num_explicit", ctypes.c_int64),
                ("resized_height", ctypes.c_int32), ("resized_width", ctypes.c_int32),
                ("image_mean", ctypes.c_float * 3), ("image_std", ctypes.c_float * 3),
                ("rescale_factor", ctypes.c_double), ("world_size", ctypes.c_int32),
                ("encoder_rank", ctypes.c_int32), ("token_dtype", ctypes.c_int), ("color", ctypes.c_int),
                ("surface_format", ctypes.c_int), ("backend", ctypes.c_int)]


class PagedTokensC(ctypes.Structure):
    _fields_ = [("pool", ctypes.c_void_p), ("pool_pages", ctypes.c_int64), ("page_rows", ctypes.c_int32),
                ("num_pages", ctypes.c_int32), ("page_ids", ctypes.POINTER(ctypes.c_int32)),
                ("first_offset", ctypes.c_int64)]


class RaggedIndexC(ctypes.Structure):
    _fields_ = [("num_requests", ctypes.c_int32), ("pv_indptr", ctypes.POINTER(ctypes.c_int64)),
                ("pv_page_indptr", ctypes.POINTER(ctypes.c_int32)),
                ("pv_page_indices", ctypes.POINTER(ctypes.c_int32)),
                ("pv_cu_page_len", ctypes.POINTER(ctypes.c_int64))]


PAGE_OPS = {"write": 0, "read": 1}


class PlanInfoC(ctypes.Structure):
    _fields_ = [("grid_thw", ctypes.c_int64 * 3), ("resized_h", ctypes.c_int32), ("resized_w", ctypes.c_int32),
                ("num_sampled", ctypes.c_int64), ("pad_frames", ctypes.c_int64), ("token_rows", ctypes.c_int64),
                ("token_cols", ctypes.c_int64), ("sampled_fps", ctypes.c_double),
                ("second_per_grid", ctypes.c_double), ("ranks_used", ctypes.c_int32),
                ("world_size", ctypes.c_int32), ("max_taps_h", ctypes.c_int32), ("max_taps_v", ctypes.c_int32)]


class RankPlanC(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("gop_begin", "gop_end", "tail_gop", "tail_frame", "sampled_begin",
                                              "sampled_count", "pad_frames", "row_begin", "row_end",
                                              "est_decode_frames")]


class TransferC(ctypes.Structure):
    _fields_ = [("peer", ctypes.c_int32), ("dir", ctypes.c_int32), ("src_offset", ctypes.c_int64),
                ("dst_offset", ctypes.c_int64), ("bytes", ctypes.c_int64)]


XCHG = {"gather": 0, "colsplit": 1}
XFER_DIRS = {0: "local", 1: "send", 2: "recv"}
KERNELS = {0: None, 1: "tc", 2: "mma"}


class Nv12SurfaceC(ctypes.Structure):
    _fields_ = [("y", ctypes.c_void_p), ("uv", ctypes.c_void_p), ("pitch_y", ctypes.c_int64),
                ("pitch_uv", ctypes.c_int64), ("v", ctypes.c_void_p)]


EXPORTS = ["fc_model_cfg_default", "fc_plan", "fc_plan_destroy", "fc_plan_info_get", "fc_plan_sampled_indices",
           "fc_plan_rank", "fc_preprocess", "fc_preprocess_debug", "fc_preprocess_batch", "fc_nccl_unique_id",
           "fc_nccl_comm_init", "fc_nccl_comm_destroy", "fc_gather", "fc_status_string", "fc_last_error",
           "fc_abi_version", "fc_kernel_launches", "fc_expand_tokens", "fc_preprocess_paged",
           "fc_preprocess_colsplit", "fc_scatter_columns", "fc_exchange_schedule", "fc_last_kernel",
           "fc_assign_requests", "fc_submit", "fc_ipc_export", "fc_ipc_export_range", "fc_ipc_import",
           "fc_ipc_close", "fc_pages_create", "fc_pages_destroy", "fc_pages_alloc", "fc_pages_index",
           "fc_pages_free_consumed", "fc_pages_release", "fc_pages_stats", "fc_paged_copy",
           "fc_jpeg_decoder_create", "fc_jpeg_decoder_destroy", "fc_jpeg_decoder_backend", "fc_jpeg_info",
           "fc_jpeg_decode_i420", "fc_dispatch_segments", "fc_decode_mjpeg"]
SEGMENT_FN = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32)
JPEG_BACKENDS = {"auto": 0, "hardware": 1, "cuda": 2}

_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                          f"g.build()'` (there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    L.fc_model_cfg_default.argtypes = [ctypes.POINTER(ModelCfgC)]
    L.fc_model_cfg_default.restype = None
    L.fc_plan.argtypes = [ctypes.POINTER(VideoMetaC), ctypes.POINTER(ModelCfgC), ctypes.POINTER(vp)]
    L.fc_plan_destroy.argtypes = [vp]
    L.fc_plan_destroy.restype = None
    L.fc_plan_info_get.argtypes = [vp, ctypes.POINTER(PlanInfoC)]
    L.fc_plan_sampled_indices.argtypes = [vp, ctypes.POINTER(ctypes.c_int64)]
    L.fc_plan_rank.argtypes = [vp, i32, ctypes.POINTER(RankPlanC)]
    L.fc_preprocess.argtypes = [vp, i32, ctypes.POINTER(Nv12SurfaceC), i64, vp, ctypes.POINTER(ctypes.c_int64), vp]
    L.fc_preprocess_debug.argtypes = [vp, i32, ctypes.POINTER(Nv12SurfaceC), i64, vp, ctypes.POINTER(ctypes.c_int64),
                                      vp, vp, vp]
    L.fc_preprocess_batch.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(ctypes.c_int32), i32,
                                      ctypes.POINTER(ctypes.POINTER(Nv12SurfaceC)), ctypes.POINTER(ctypes.c_int64),
                                      ctypes.POINTER(vp), vp]
    L.fc_nccl_unique_id.argtypes = [ctypes.POINTER(ctypes.c_uint8)]
    L.fc_nccl_comm_init.argtypes = [ctypes.POINTER(ctypes.c_uint8), i32, i32, ctypes.POINTER(vp)]
    L.fc_nccl_comm_destroy.argtypes = [vp]
    L.fc_gather.argtypes = [vp, i32, vp, vp, vp, vp]
    L.fc_preprocess_colsplit.argtypes = [vp, i32, ctypes.POINTER(Nv12SurfaceC), i64, vp, ctypes.POINTER(i64), vp]
    L.fc_scatter_columns.argtypes = [vp, i32, vp, vp, vp, vp]
    L.fc_status_string.argtypes = [ctypes.c_int]
    L.fc_status_string.restype = ctypes.c_char_p
    L.fc_last_error.argtypes = []
    L.fc_last_error.restype = ctypes.c_char_p
    L.fc_abi_version.argtypes = []
    L.fc_abi_version.restype = ctypes.c_int32
    L.fc_expand_tokens.argtypes = [vp, i64, vp, vp, ctypes.c_int, vp]
    L.fc_preprocess_paged.argtypes = [vp, i32, ctypes.POINTER(Nv12SurfaceC), i64, ctypes.POINTER(PagedTokensC),
                                      ctypes.POINTER(ctypes.c_int64), vp]
    L.fc_kernel_launches.argtypes = []
    L.fc_kernel_launches.restype = ctypes.c_uint64
    L.fc_exchange_schedule.argtypes = [vp, i32, ctypes.c_int, ctypes.POINTER(TransferC), i32, ctypes.POINTER(i32)]
    L.fc_assign_requests.argtypes = [ctypes.POINTER(ctypes.c_int64), i32, i32, ctypes.POINTER(ctypes.c_int32)]
    L.fc_submit.argtypes = [ctypes.POINTER(VideoMetaC), ctypes.POINTER(ModelCfgC), i32, ctypes.POINTER(Nv12SurfaceC),
                            i64, vp, vp, ctypes.POINTER(vp)]
    L.fc_ipc_export.argtypes = [vp, ctypes.POINTER(ctypes.c_uint8)]
    L.fc_ipc_export_range.argtypes = [vp, ctypes.POINTER(ctypes.c_uint8), ctypes.POINTER(ctypes.c_int64)]
    L.fc_ipc_import.argtypes = [ctypes.POINTER(ctypes.c_uint8), ctypes.POINTER(vp)]
    L.fc_ipc_close.argtypes = [vp]
    pi32, pi64 = ctypes.POINTER(i32), ctypes.POINTER(i64)
    L.fc_pages_create.argtypes = [i64, i32, ctypes.POINTER(vp)]
    L.fc_pages_destroy.argtypes = [vp]
    L.fc_pages_destroy.restype = None
    L.fc_pages_alloc.argtypes = [vp, i64, i64, pi32, i32, pi32]
    L.fc_pages_index.argtypes = [vp, ctypes.c_int, pi64, pi64, i32, pi64, pi32, pi32, i32, pi64, pi32]
    L.fc_pages_free_consumed.argtypes = [vp, pi32, i32, pi32]
    L.fc_pages_release.argtypes = [vp, i64]
    L.fc_pages_stats.argtypes = [vp, pi64, pi64, pi64, pi64]
    L.fc_paged_copy.argtypes = [ctypes.c_int, ctypes.POINTER(RaggedIndexC), vp, i64, i32, i64, vp, vp]
    L.fc_last_kernel.argtypes = []
    L.fc_last_kernel.restype = ctypes.c_int32
    L.fc_jpeg_decoder_create.argtypes = [i32, ctypes.POINTER(vp)]
    L.fc_jpeg_decoder_destroy.argtypes = [vp]
    L.fc_jpeg_decoder_destroy.restype = None
    L.fc_jpeg_decoder_backend.argtypes = [vp]
    L.fc_jpeg_decoder_backend.restype = ctypes.c_int32
    L.fc_jpeg_info.argtypes = [vp, ctypes.c_char_p, ctypes.c_size_t, pi32, pi32, pi32]
    L.fc_jpeg_decode_i420.argtypes = [vp, ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(Nv12SurfaceC), vp]
    L.fc_dispatch_segments.argtypes = [ctypes.POINTER(ctypes.c_int32), i64, i32, i32, SEGMENT_FN, vp,
                                       ctypes.POINTER(ctypes.c_int64)]
    L.fc_decode_mjpeg.argtypes = [ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_size_t), i64,
                                  ctypes.POINTER(Nv12SurfaceC), i32, i32, i32, i32, ctypes.POINTER(ctypes.c_int64)]
    for name in EXPORTS:
        fn = getattr(L, name)
        if name not in ("fc_model_cfg_default", "fc_plan_destroy", "fc_pages_destroy", "fc_status_string", "fc_last_error",
                        "fc_abi_version", "fc_kernel_launches", "fc_last_kernel", "fc_jpeg_decoder_destroy",
                        "fc_jpeg_decoder_backend"):
            fn.restype = ctypes.c_int
    _lib = L
    return L


def check(status: int, where: str) -> None:
    if status != 0:
        detail = lib().fc_last_error().decode(errors="replace")
        raise FcError(status, where, detail)
