"""B200-native FlashCodec preprocessing hot path (arXiv 2512.17574).

Thin Python binding over the C ABI in ``include/fc.h`` (``libfc.so``):
argument marshalling only -- every step of the path runs in the library's
sm_100a kernels / host planner.  PyTorch is used for device memory, streams
and process groups.

    meta = VideoMeta(1920, 1080, 1800, fps=(30, 1), gop_start=range(0, 1800, 30))
    plan = Plan(meta, ModelCfg(world_size=1))            # fc_plan
    surf = SurfaceTable.from_tensors(ys, uvs)            # fc_nv12_surface[]
    tokens = preprocess(plan, 0, surf)                   # fc_preprocess
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from fractions import Fraction
from typing import Sequence

from . import _native
from ._native import FcError, FC_TOKEN_COLS, check, lib

__all__ = ["VideoMeta", "ModelCfg", "Plan", "SurfaceTable", "preprocess", "preprocess_debug", "preprocess_batch",
           "expand_tokens", "preprocess_paged", "PageTable", "RaggedIndex", "paged_copy",
           "NcclComm", "gather", "exchange_schedule", "last_kernel", "assign_requests", "submit", "ipc_export", "PeerBuffer", "FcError", "FC_TOKEN_COLS", "lib",
           "JpegDecoder", "image_cfg", "preprocess_jpeg", "dispatch_segments", "decode_mjpeg"]


@dataclass
class VideoMeta:
    """Video metadata M (Alg. 1 l.2): luma size, frame count,
    frame rate (rational), GOP start indices (presentation order)."""
    width: int
    height: int
    num_frames: int
    fps: tuple[int, int] | Fraction | int = (30, 1)
    gop_start: Sequence[int] = (0,)

    def to_c(self):
        # requests of one shape reuse the marshalled struct (keyed by every field)
        key = (self.width, self.height, self.num_frames, self.fps, tuple(self.gop_start))
        cached = self.__dict__.get("_c")
        if cached is not None and cached[0] == key:
            return cached[1], cached[2]
        m, arr = self._to_c()
        self.__dict__["_c"] = (key, m, arr)
        return m, arr

    def _to_c(self):
        fr = Fraction(self.fps[0], self.fps[1]) if isinstance(self.fps, tuple) else Fraction(self.fps)
        gs = list(self.gop_start)
        arr = (ctypes.c_int64 * len(gs))(*gs)
        m = _native.VideoMetaC(self.width, self.height, self.num_frames, _native.Rational(fr.numerator, fr.denominator),
                               len(gs), ctypes.cast(arr, ctypes.POINTER(ctypes.c_int64)))
        return m, arr


@dataclass
class ModelCfg:
    """Preprocessing configuration; defaults = Qwen2-VL video processor (R1, R2, R5)."""
    world_size: int = 1
    encoder_rank: int = 0
    sampling: str = "fps_stride"
    sample_fps: float = 2.0
    num_frames: int = 0
    min_frames: int = 4
    max_frames: int = 768
    explicit_indices: Sequence[int] | None = None
    min_pixels: int = 128 * 28 * 28
    max_pixels: int = 768 * 28 * 28
    total_pixels: float = 0.0
    resized_height: int = 0
    resized_width: int = 0
    image_mean: tuple[float, float, float] | None = None
    image_std: tuple[float, float, float] | None = None
    rescale_factor: float | None = None
    token_dtype: str = "f32"        # "f32" (HF output) | "bf16" (R16) | "u8" (codes; NEXT-1 exchange format)
    color: str = "bt601"            # "bt601" (R3) | "bt709" | "bt601_full" | "bt709_full" (R15)
    surface_format: str = "nv12"    # "nv12" (interleaved chroma) | "i420" (planar U, V)
    backend: str = "pil"            # HF processor arithmetic (R21): "pil" | "torchvision" (CPU uint8 AA bicubic)

    def to_c(self):
        key = tuple(tuple(v) if isinstance(v, (list, tuple)) else v for k, v in self.__dict__.items() if k != "_c")
        cached = self.__dict__.get("_c")
        if cached is not None and cached[0] == key:
            return cached[1], cached[2]
        c, keep = self._to_c()
        self.__dict__["_c"] = (key, c, keep)
        return c, keep

    def _to_c(self):
        c = _native.ModelCfgC()
        lib().fc_model_cfg_default(ctypes.byref(c))
        c.world_size = self.world_size
        c.encoder_rank = self.encoder_rank
        c.sampling = _native.SAMPLING[self.sampling]
        c.token_dtype = _native.TOKEN_DTYPES[self.token_dtype]
        c.color = _native.COLORS[self.color]
        c.surface_format = _native.SURFACES[self.surface_format]
        c.backend = _native.BACKENDS[self.backend]
        c.sample_fps = self.sample_fps
        c.num_frames = self.num_frames
        c.min_frames = self.min_frames
        c.max_frames = self.max_frames
        c.min_pixels = self.min_pixels
        c.max_pixels = self.max_pixels
        c.total_pixels = self.total_pixels
        c.resized_height = self.resized_height
        c.resized_width = self.resized_width
        if self.image_mean is not None:
            c.image_mean = (ctypes.c_float * 3)(*self.image_mean)
        if self.image_std is not None:
            c.image_std = (ctypes.c_float * 3)(*self.image_std)
        if self.rescale_factor is not None:
            c.rescale_factor = self.rescale_factor
        keep = None
        if self.explicit_indices is not None:
            keep = (ctypes.c_int64 * len(self.explicit_indices))(*self.explicit_indices)
            c.explicit_indices = ctypes.cast(keep, ctypes.POINTER(ctypes.c_int64))
            c.num_explicit = len(self.explicit_indices)
        return c, keep


class Plan:
    """fc_plan: sampling + smart_resize + GOP->rank partition + tables (host)."""

    def __init__(self, meta: VideoMeta, cfg: ModelCfg | None = None, _handle=None):
        self.meta = meta
        self.cfg = cfg or ModelCfg()
        if _handle is None:
            m, _keep_m = meta.to_c()
            c, _keep_c = self.cfg.to_c()
            h = ctypes.c_void_p()
            check(lib().fc_plan(ctypes.byref(m), ctypes.byref(c), ctypes.byref(h)), "fc_plan")
        else:  # a plan created by fc_submit
            h = _handle
        self._h = h
        info = _native.PlanInfoC()
        check(lib().fc_plan_info_get(h, ctypes.byref(info)), "fc_plan_info_get")
        self.grid_thw = tuple(info.grid_thw)
        self.resized = (info.resized_h, info.resized_w)
        self.num_sampled = info.num_sampled
        self.pad_frames = info.pad_frames
        self.token_rows = info.token_rows
        self.sampled_fps = info.sampled_fps
        self.second_per_grid = info.second_per_grid
        self.ranks_used = info.ranks_used
        self.world_size = info.world_size
        self.max_taps = (info.max_taps_h, info.max_taps_v)
        self._sampled = None
        self._rows: dict[int, int] = {}

    @property
    def sampled_indices(self) -> list[int]:
        """fc_plan_sampled_indices (fetched on first use)."""
        if self._sampled is None:
            idx = (ctypes.c_int64 * max(self.num_sampled, 1))()
            check(lib().fc_plan_sampled_indices(self._h, idx), "fc_plan_sampled_indices")
            self._sampled = list(idx)[: self.num_sampled]
        return self._sampled

    def rank_rows(self, r: int) -> int:
        """Token rows of rank r (row_end - row_begin; the plan is immutable, so cached)."""
        n = self._rows.get(r)
        if n is None:
            rp = self.rank(r)
            n = self._rows[r] = rp["row_end"] - rp["row_begin"]
        return n

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    def rank(self, r: int) -> dict:
        rp = _native.RankPlanC()
        check(lib().fc_plan_rank(self._h, r, ctypes.byref(rp)), "fc_plan_rank")
        return {n: getattr(rp, n) for n, _ in rp._fields_}

    def ranks(self) -> list[dict]:
        return [self.rank(r) for r in range(self.world_size)]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                lib().fc_plan_destroy(h)
            except TypeError:  # interpreter teardown: module globals already cleared
                pass
            self._h = None


class SurfaceTable:
    """A host array of fc_nv12_surface descriptors, indexed by GLOBAL frame
    index (entries a rank does not read may be empty).  Holds references to
    the tensors so they stay alive."""

    def __init__(self, num_frames: int):
        self.arr = (_native.Nv12SurfaceC * max(num_frames, 1))()
        self.n = num_frames
        self._keep: dict[int, tuple] = {}

    def set(self, frame: int, y, uv, v=None) -> None:
        """NV12: y uint8 [H, pitch_y] device tensor, uv uint8 [H/2, pitch_uv]
        (interleaved U,V).  I420: uv = the U plane and v = the V plane, both
        uint8 [H/2, pitch_uv] (same pitch)."""
        if v is not None and v.stride(0) != uv.stride(0):
            raise ValueError("I420 U and V planes must share the pitch")
        self.arr[frame] = _native.Nv12SurfaceC(y.data_ptr(), uv.data_ptr(), y.stride(0), uv.stride(0),
                                               v.data_ptr() if v is not None else None)
        self._keep[frame] = (y, uv, v)

    @classmethod
    def from_tensors(cls, frames: dict | Sequence, num_frames: int | None = None) -> "SurfaceTable":
        items = frames.items() if isinstance(frames, dict) else enumerate(frames)
        items = list(items)
        n = num_frames if num_frames is not None else (max(k for k, _ in items) + 1 if items else 0)
        t = cls(n)
        for k, v in items:
            if v is not None:
                t.set(k, *v)
        return t


def _stream_ptr(stream) -> ctypes.c_void_p:
    import torch
    if stream is None:  # the current stream's handle, without building a Stream object
        return ctypes.c_void_p(torch._C._cuda_getCurrentRawStream(torch.cuda.current_device()))
    return ctypes.c_void_p(stream.cuda_stream)


def _tok_dtype(plan: Plan):
    import torch
    return {"f32": torch.float32, "bf16": torch.bfloat16, "u8": torch.uint8}[plan.cfg.token_dtype]


def _rank_rows(plan: Plan, rank: int) -> int:
    return plan.rank_rows(rank)


def preprocess(plan: Plan, rank: int, surfaces: SurfaceTable, out=None, stream=None):
    """fc_preprocess: enqueue the fused kernel for `rank` on `stream`; returns
    the (row_end-row_begin) x 1176 fp32 token shard (allocated after planning
    if `out` is None)."""
    import torch
    if out is None:
        out = torch.empty((_rank_rows(plan, rank), FC_TOKEN_COLS), dtype=_tok_dtype(plan), device="cuda")
    check(lib().fc_preprocess(plan.handle, rank, surfaces.arr, surfaces.n, ctypes.c_void_p(out.data_ptr()), None,
                              _stream_ptr(stream)), "fc_preprocess")
    return out


def submit(meta: VideoMeta, cfg: ModelCfg, rank: int, surfaces: SurfaceTable, out, stream=None) -> Plan:
    """fc_submit: plan the request and enqueue its fused kernel in ONE C call
    (small requests, where per-call overhead dominates); `out` is the
    caller-allocated token shard of `rank`.  Returns the request's Plan."""
    m, _km = meta.to_c()
    c, _kc = cfg.to_c()
    h = ctypes.c_void_p()
    check(lib().fc_submit(ctypes.byref(m), ctypes.byref(c), rank, surfaces.arr, surfaces.n,
                          ctypes.c_void_p(out.data_ptr()), _stream_ptr(stream), ctypes.byref(h)), "fc_submit")
    return Plan(meta, cfg, _handle=h)


def preprocess_debug(plan: Plan, rank: int, surfaces: SurfaceTable, stream=None):
    """fc_preprocess_debug: tokens plus the integer intermediates
    (BT.601 RGB [n_r,H,W,3] and resized RGB [n_r,H',W',3], u8)."""
    import torch
    rp = plan.rank(rank)
    rows = rp["row_end"] - rp["row_begin"]
    nr = rp["sampled_count"] + rp["pad_frames"]
    h2, w2 = plan.resized
    tokens = torch.empty((rows, FC_TOKEN_COLS), dtype=torch.float32, device="cuda")
    src = torch.empty((nr, plan.meta.height, plan.meta.width, 3), dtype=torch.uint8, device="cuda")
    rs = torch.empty((nr, h2, w2, 3), dtype=torch.uint8, device="cuda")
    grid = (ctypes.c_int64 * 3)()
    check(lib().fc_preprocess_debug(plan.handle, rank, surfaces.arr, surfaces.n, ctypes.c_void_p(tokens.data_ptr()),
                                    grid, _stream_ptr(stream), ctypes.c_void_p(src.data_ptr()),
                                    ctypes.c_void_p(rs.data_ptr())), "fc_preprocess_debug")
    return tokens, src, rs


def preprocess_batch(jobs: Sequence[tuple[Plan, int, SurfaceTable]], outs=None, stream=None):
    """fc_preprocess_batch: several independent (plan, rank) jobs on one stream;
    consecutive jobs of equal geometry and pair count share ONE launch (a
    config-5 batch of same-shape clips is a single persistent launch)."""
    import torch
    n = len(jobs)
    if outs is None:
        outs = [torch.empty((_rank_rows(p, r), FC_TOKEN_COLS), dtype=_tok_dtype(p), device="cuda")
                for p, r, _ in jobs]
    plans = (ctypes.c_void_p * n)(*[p.handle.value for p, _, _ in jobs])
    ranks = (ctypes.c_int32 * n)(*[r for _, r, _ in jobs])
    surfs = (ctypes.POINTER(_native.Nv12SurfaceC) * n)(*[ctypes.cast(s.arr, ctypes.POINTER(_native.Nv12SurfaceC))
                                                         for _, _, s in jobs])
    nsurf = (ctypes.c_int64 * n)(*[s.n for _, _, s in jobs])
    toks = (ctypes.c_void_p * n)(*[o.data_ptr() for o in outs])
    check(lib().fc_preprocess_batch(plans, ranks, n, surfs, nsurf, toks, _stream_ptr(stream)), "fc_preprocess_batch")
    return outs


def preprocess_paged(plan: Plan, rank: int, surfaces: SurfaceTable, pool, page_ids: Sequence[int],
                     first_offset: int = 0, stream=None) -> None:
    """fc_preprocess_paged (NEXT-2): write the rank's token rows, in order, as
    one write chunk of a paged buffer.  pool: device tensor [pool_pages,
    page_rows, 1176] of the plan's token dtype; page_ids: this write's pages
    (pv_page_indices segment); first_offset: pv_cu_page_len mod page_rows."""
    ids = (ctypes.c_int32 * max(len(page_ids), 1))(*page_ids)
    d = _native.PagedTokensC(ctypes.c_void_p(pool.data_ptr()), pool.shape[0], pool.shape[1], len(page_ids),
                             ctypes.cast(ids, ctypes.POINTER(ctypes.c_int32)), first_offset)
    grid = (ctypes.c_int64 * 3)()
    check(lib().fc_preprocess_paged(plan.handle, rank, surfaces.arr, surfaces.n, ctypes.byref(d), grid,
                                    _stream_ptr(stream)), "fc_preprocess_paged")


@dataclass
class RaggedIndex:
    """One iteration's four indices: pv_indptr [n+1],
    pv_page_indptr [n+1], pv_page_indices, pv_cu_page_len [n] (host lists)."""
    pv_indptr: list
    pv_page_indptr: list
    pv_page_indices: list
    pv_cu_page_len: list

    def to_c(self):
        n = len(self.pv_cu_page_len)
        arrs = ((ctypes.c_int64 * (n + 1))(*self.pv_indptr), (ctypes.c_int32 * (n + 1))(*self.pv_page_indptr),
                (ctypes.c_int32 * max(len(self.pv_page_indices), 1))(*self.pv_page_indices),
                (ctypes.c_int64 * max(n, 1))(*self.pv_cu_page_len))
        c = _native.RaggedIndexC(n, *(ctypes.cast(a, ctypes.POINTER(t)) for a, t in
                                      zip(arrs, (ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64))))
        return c, arrs  # keep arrs alive with the struct


class PageTable:
    """fc_pages_* (NEXT-2): the paged embedding buffer's page table
    (host bookkeeping in libfc; the data moves in fc_preprocess_paged and
    fc_paged_copy)."""

    def __init__(self, total_pages: int, page_rows: int):
        self._h = ctypes.c_void_p()
        check(lib().fc_pages_create(total_pages, page_rows, ctypes.byref(self._h)), "fc_pages_create")
        self.total_pages, self.page_rows = total_pages, page_rows

    def alloc(self, req: int, tokens: int) -> list[int]:
        cap = tokens // self.page_rows + 2
        ids, n = (ctypes.c_int32 * cap)(), ctypes.c_int32()
        check(lib().fc_pages_alloc(self._h, req, tokens, ids, cap, ctypes.byref(n)), "fc_pages_alloc")
        return list(ids[:n.value])

    def index(self, op: str, reqs: Sequence[int], counts: Sequence[int]) -> RaggedIndex:
        n = len(reqs)
        r, c = (ctypes.c_int64 * max(n, 1))(*reqs), (ctypes.c_int64 * max(n, 1))(*counts)
        indptr, pindptr, cu = (ctypes.c_int64 * (n + 1))(), (ctypes.c_int32 * (n + 1))(), (ctypes.c_int64 * max(n, 1))()
        m = ctypes.c_int32()
        cap = sum(int(x) // self.page_rows + 2 for x in counts)
        pages = (ctypes.c_int32 * max(cap, 1))()
        check(lib().fc_pages_index(self._h, _native.PAGE_OPS[op], r, c, n, indptr, pindptr, pages, cap, cu,
                                   ctypes.byref(m)), "fc_pages_index")
        return RaggedIndex(list(indptr), list(pindptr), list(pages[:m.value]), list(cu[:n]))

    def free_consumed(self) -> list[int]:
        _, _, consumed, _ = self.stats()
        ids, n = (ctypes.c_int32 * max(consumed, 1))(), ctypes.c_int32()
        check(lib().fc_pages_free_consumed(self._h, ids, max(consumed, 1), ctypes.byref(n)), "fc_pages_free_consumed")
        return list(ids[:n.value])

    def release(self, req: int) -> None:
        check(lib().fc_pages_release(self._h, req), "fc_pages_release")

    def stats(self) -> tuple[int, int, int, int]:
        """(free pages, owned pages, consumed pages, live requests)"""
        v = [ctypes.c_int64() for _ in range(4)]
        check(lib().fc_pages_stats(self._h, *(ctypes.byref(x) for x in v)), "fc_pages_stats")
        return tuple(x.value for x in v)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().fc_pages_destroy(h)
            except (TypeError, AttributeError):  # interpreter teardown: module globals already cleared
                pass
            self._h = None


def paged_copy(op: str, index: RaggedIndex, pool, chunk, stream=None) -> None:
    """fc_paged_copy (NEXT-2 read_chunk / write_chunk): op "read" gathers the
    iteration's tokens from pool [pool_pages, page_rows, cols] into chunk
    [pv_indptr[-1], cols]; "write" scatters them back.  One HBM-bound launch."""
    c, _keep = index.to_c()
    row_bytes = pool.shape[2] * pool.element_size()
    check(lib().fc_paged_copy(_native.PAGE_OPS[op], ctypes.byref(c), ctypes.c_void_p(pool.data_ptr()), pool.shape[0],
                              pool.shape[1], row_bytes, ctypes.c_void_p(chunk.data_ptr()), _stream_ptr(stream)),
          "fc_paged_copy")


def expand_tokens(plan: Plan, codes, out=None, out_dtype: str = "f32", stream=None):
    """fc_expand_tokens: u8 codes [rows, 1176] -> f32/bf16 tokens with the
    plan's normalisation (one HBM-bound launch)."""
    import torch
    rows = codes.shape[0]
    if out is None:
        out = torch.empty((rows, FC_TOKEN_COLS), dtype=torch.bfloat16 if out_dtype == "bf16" else torch.float32,
                          device="cuda")
    check(lib().fc_expand_tokens(plan.handle, rows, ctypes.c_void_p(codes.data_ptr()),
                                 ctypes.c_void_p(out.data_ptr()), _native.TOKEN_DTYPES[out_dtype],
                                 _stream_ptr(stream)), "fc_expand_tokens")
    return out


class NcclComm:
    """An NCCL communicator owned by libfc (fc_nccl_comm_init), bootstrapped
    over an existing torch.distributed process group (the 128-byte unique id
    is broadcast with it)."""

    def __init__(self, rank: int, world_size: int, group=None):
        import torch
        import torch.distributed as dist
        idbuf = (ctypes.c_uint8 * 128)()
        if rank == 0:
            check(lib().fc_nccl_unique_id(idbuf), "fc_nccl_unique_id")
        t = torch.tensor(list(bytes(idbuf)), dtype=torch.uint8)
        backend = dist.get_backend(group)
        if backend == "nccl":
            t = t.cuda()
        dist.broadcast(t, src=0, group=group)
        idbuf = (ctypes.c_uint8 * 128)(*t.cpu().tolist())
        h = ctypes.c_void_p()
        check(lib().fc_nccl_comm_init(idbuf, world_size, rank, ctypes.byref(h)), "fc_nccl_comm_init")
        self.handle = h

    def close(self):
        if self.handle:
            check(lib().fc_nccl_comm_destroy(self.handle), "fc_nccl_comm_destroy")
            self.handle = None


def preprocess_colsplit(plan: Plan, rank: int, surfaces: SurfaceTable, out=None, stream=None):
    """fc_preprocess_colsplit (NEXT-1): the rank's tokens as W column
    blocks, fp32 [W, rows_r, 1176 // W]."""
    import torch
    w = plan.cfg.world_size
    rows = _rank_rows(plan, rank)
    if out is None:
        out = torch.empty((w, rows, FC_TOKEN_COLS // w), dtype=torch.float32, device="cuda")
    grid = (ctypes.c_int64 * 3)()
    check(lib().fc_preprocess_colsplit(plan.handle, rank, surfaces.arr, surfaces.n, ctypes.c_void_p(out.data_ptr()),
                                       grid, _stream_ptr(stream)), "fc_preprocess_colsplit")
    return out


def scatter_columns(plan: Plan, rank: int, comm: NcclComm | None, blocks, mine=None, stream=None):
    """fc_scatter_columns: all-to-all of the column blocks; returns this rank's
    column slice of every token row, fp32 [token_rows, 1176 // W]."""
    import torch
    w = plan.cfg.world_size
    if mine is None:
        mine = torch.empty((plan.token_rows, FC_TOKEN_COLS // w), dtype=torch.float32, device="cuda")
    check(lib().fc_scatter_columns(plan.handle, rank, comm.handle if comm else None,
                                   ctypes.c_void_p(blocks.data_ptr()) if blocks is not None else None,
                                   ctypes.c_void_p(mine.data_ptr()), _stream_ptr(stream)), "fc_scatter_columns")
    return mine


def exchange_schedule(plan: Plan, rank: int, kind: str = "gather") -> list[dict]:
    """fc_exchange_schedule: the transfers `rank` issues in fc_gather
    (kind="gather") or fc_scatter_columns (kind="colsplit"), as dicts
    {peer, dir ("local" | "send" | "recv"), src_offset, dst_offset, bytes}."""
    n = ctypes.c_int32()
    check(lib().fc_exchange_schedule(plan.handle, rank, _native.XCHG[kind], None, 0, ctypes.byref(n)),
          "fc_exchange_schedule")
    arr = (_native.TransferC * max(n.value, 1))()
    check(lib().fc_exchange_schedule(plan.handle, rank, _native.XCHG[kind], arr, n.value, ctypes.byref(n)),
          "fc_exchange_schedule")
    return [dict(peer=t.peer, dir=_native.XFER_DIRS[t.dir], src_offset=t.src_offset, dst_offset=t.dst_offset,
                 bytes=t.bytes) for t in arr[: n.value]]


def assign_requests(pairs: Sequence[int], world: int) -> list[int]:
    """fc_assign_requests: GPU of each whole request (LPT on temporal pairs;
    throughput mode, no exchange)."""
    n = len(pairs)
    arr = (ctypes.c_int64 * max(n, 1))(*pairs)
    out = (ctypes.c_int32 * max(n, 1))()
    check(lib().fc_assign_requests(arr, n, world, out), "fc_assign_requests")
    return list(out)[:n]


def ipc_export(tensor) -> tuple[bytes, int]:
    """fc_ipc_export_range: (64-byte IPC handle of the allocation holding
    `tensor`, byte offset of tensor.data_ptr() in it) -- for another process
    to map (ipc_import) and write into (the fused peer-store exchange)."""
    h = (ctypes.c_uint8 * 64)()
    off = ctypes.c_int64()
    check(lib().fc_ipc_export_range(ctypes.c_void_p(tensor.data_ptr()), h, ctypes.byref(off)), "fc_ipc_export_range")
    return bytes(h), off.value


class PeerBuffer:
    """A peer process's device buffer mapped into this process
    (fc_ipc_import); `tensor(shape, dtype, offset)` views it as a torch
    tensor (no copy; writes land in the peer's memory).  close() unmaps."""

    def __init__(self, handle: bytes):
        p = ctypes.c_void_p()
        check(lib().fc_ipc_import((ctypes.c_uint8 * 64)(*handle), ctypes.byref(p)), "fc_ipc_import")
        self.ptr = p.value

    def tensor(self, shape, dtype, offset: int = 0):
        import torch

        class _View:  # __cuda_array_interface__ (v3) for torch.as_tensor
            def __init__(self, ptr, shape, typestr):
                self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                                 "version": 3, "strides": None}
        typestr = {torch.float32: "<f4", torch.bfloat16: "<V2", torch.uint8: "|u1"}[dtype]
        if dtype == torch.bfloat16:  # no bf16 typestr: view the bytes as int16 and reinterpret
            t = torch.as_tensor(_View(self.ptr + offset, shape, "<i2"), device="cuda")
            return t.view(torch.bfloat16)
        return torch.as_tensor(_View(self.ptr + offset, shape, typestr), device="cuda")

    def close(self):
        if self.ptr:
            check(lib().fc_ipc_close(ctypes.c_void_p(self.ptr)), "fc_ipc_close")
            self.ptr = None


def last_kernel() -> str | None:
    """fc_last_kernel: "tc" (tcgen05 kernel) or "mma" (mma.sync kernel) for
    this thread's last fc_preprocess* launch."""
    return _native.KERNELS[lib().fc_last_kernel()]


def gather(plan: Plan, rank: int, comm: NcclComm | None, shard, full=None, stream=None):
    """fc_gather: gatherv of the row shards into the encoder rank's full
    token buffer (returned on the encoder rank, None elsewhere)."""
    import torch
    enc = plan.cfg.encoder_rank
    if rank == enc and full is None:
        full = torch.empty((plan.token_rows, FC_TOKEN_COLS), dtype=_tok_dtype(plan), device="cuda")
    check(lib().fc_gather(plan.handle, rank, comm.handle if comm else None,
                          ctypes.c_void_p(shard.data_ptr()) if shard is not None else None,
                          ctypes.c_void_p(full.data_ptr()) if full is not None else None,
                          _stream_ptr(stream)), "fc_gather")
    return full if rank == enc else None


# ---------------------------------------------------------------- JPEG images
class JpegDecoder:
    """NEXT-4 image path ("JPEG is decoded via dedicated hardware"):
    nvJPEG (hardware engines when offered, else its CUDA decoder) decodes a
    4:2:0 JPEG into device I420 planes that the fused kernel consumes like a
    decoded video frame (fc.h fc_jpeg_*)."""

    def __init__(self, backend: str = "auto"):
        h = ctypes.c_void_p()
        check(lib().fc_jpeg_decoder_create(_native.JPEG_BACKENDS[backend], ctypes.byref(h)), "fc_jpeg_decoder_create")
        self.handle = h
        # why the hardware backend was not taken (auto mode), from the library's last error
        self.hardware_error = (lib().fc_last_error().decode(errors="replace")
                               if backend == "auto" and lib().fc_jpeg_decoder_backend(h) != 1 else "")

    @property
    def backend(self) -> str:
        return {1: "hardware", 2: "cuda"}[lib().fc_jpeg_decoder_backend(self.handle)]

    def info(self, data: bytes) -> tuple[int, int, bool]:
        w, h, css = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        check(lib().fc_jpeg_info(self.handle, data, len(data), ctypes.byref(w), ctypes.byref(h), ctypes.byref(css)),
              "fc_jpeg_info")
        return w.value, h.value, css.value == 0

    def decode(self, data: bytes, stream=None):
        """-> (y [H, pitch], u [H/2, pitch_c], v [H/2, pitch_c]) uint8 device tensors
        (pitches rounded up to 256 bytes, NVDEC-like)."""
        import torch
        w, h, _ = self.info(data)
        py, pc = (w + 255) // 256 * 256, (w // 2 + 255) // 256 * 256
        y = torch.empty((h, py), dtype=torch.uint8, device="cuda")
        u = torch.empty((h // 2, pc), dtype=torch.uint8, device="cuda")
        v = torch.empty((h // 2, pc), dtype=torch.uint8, device="cuda")
        s = _native.Nv12SurfaceC(y.data_ptr(), u.data_ptr(), py, pc, v.data_ptr())
        check(lib().fc_jpeg_decode_i420(self.handle, data, len(data), ctypes.byref(s), _stream_ptr(stream)),
              "fc_jpeg_decode_i420")
        return y, u, v

    def close(self) -> None:
        if self.handle:
            lib().fc_jpeg_decoder_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def image_cfg(**kw) -> ModelCfg:
    """Preprocessing of a JPEG image through the video path: full-range BT.601
    (JFIF), I420 surfaces, one explicitly sampled frame (padded to the temporal
    patch); other fields as given (e.g. the image processor's pixel budget)."""
    kw.setdefault("color", "bt601_full")
    kw.setdefault("surface_format", "i420")
    kw.setdefault("sampling", "explicit")
    kw.setdefault("explicit_indices", [0])
    return ModelCfg(**kw)


def preprocess_jpeg(decoder: JpegDecoder, data: bytes, cfg: ModelCfg | None = None, stream=None):
    """One JPEG image -> (tokens [H'/14 * W'/14, 1176], grid_thw (1, H'/14, W'/14), plan)."""
    cfg = cfg or image_cfg()
    w, h, _ = decoder.info(data)
    planes = decoder.decode(data, stream)
    plan = Plan(VideoMeta(w, h, 1, (1, 1), [0]), cfg)
    surf = SurfaceTable(1)
    surf.set(0, *planes)
    tokens = preprocess(plan, 0, surf, stream=stream)
    return tokens, plan.grid_thw, plan, planes


# ------------------------------------------------- stall-free GOP_s dispatch
def dispatch_segments(worker_of: Sequence[int], num_workers: int, max_in_flight: int, fn) -> list[tuple[int, int, int]]:
    """fc_dispatch_segments (Alg. 2): run fn(segment, worker) -> int (0 = ok) on
    num_workers threads, at most max_in_flight at once, a worker keeping its
    unit for its next segment.  Returns the completion trace
    [(segment, worker, status)].  (fn runs on library threads; a Python fn
    takes the GIL per call.)"""
    n = len(worker_of)
    wo = (ctypes.c_int32 * max(n, 1))(*worker_of)
    trace = (ctypes.c_int64 * max(3 * n, 1))()

    def cb(_ctx, seg, w):
        try:
            return int(fn(int(seg), int(w)))
        except Exception:  # a raising callback is a failed segment
            return 1
    cfn = _native.SEGMENT_FN(cb)
    check(lib().fc_dispatch_segments(wo, n, num_workers, max_in_flight, cfn, None, trace), "fc_dispatch_segments")
    return [(trace[3 * i], trace[3 * i + 1], trace[3 * i + 2]) for i in range(n)]


def decode_mjpeg(frames: Sequence[bytes], segments: int = 4, workers: int = 2, max_in_flight: int = 2,
                 backend: str = "auto"):
    """fc_decode_mjpeg: the target frames of a Motion-JPEG request (each an
    independent 4:2:0 JPEG) -> a list of (y, u, v) device tensors, decoded by
    `workers` threads over GOP_s segments with at most `max_in_flight` at once
    (Alg. 2).  Returns (planes, trace)."""
    import torch
    n = len(frames)
    info = JpegDecoder(backend)
    planes, arr = [], (_native.Nv12SurfaceC * max(n, 1))()
    for i, f in enumerate(frames):
        w, h, _ = info.info(f)
        py, pc = (w + 255) // 256 * 256, (w // 2 + 255) // 256 * 256
        y = torch.empty((h, py), dtype=torch.uint8, device="cuda")
        u = torch.empty((h // 2, pc), dtype=torch.uint8, device="cuda")
        v = torch.empty((h // 2, pc), dtype=torch.uint8, device="cuda")
        arr[i] = _native.Nv12SurfaceC(y.data_ptr(), u.data_ptr(), py, pc, v.data_ptr())
        planes.append((y, u, v))
    info.close()
    data = (ctypes.c_char_p * max(n, 1))(*frames)
    lens = (ctypes.c_size_t * max(n, 1))(*[len(f) for f in frames])
    trace = (ctypes.c_int64 * max(3 * min(segments, n), 1))()
    check(lib().fc_decode_mjpeg(data, lens, n, arr, segments, workers, max_in_flight,
                                _native.JPEG_BACKENDS[backend], trace), "fc_decode_mjpeg")
    return planes, [(trace[3 * i], trace[3 * i + 1], trace[3 * i + 2]) for i in range(min(segments, n))]
