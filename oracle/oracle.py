"""CPU ORACLE for the FlashCodec preprocessing hot path -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module.  The
product package ``paper_2512_17574_b200`` never imports it; the two share no
code (only the seeded input generators in ``synth/`` serve both).

Contents, each citing what it follows (P:n = /root/reference/PAPER.md line n,
SURVEY = /root/repo/SURVEY.md; readings listed in DESIGN.md "Readings"):

* ``sample_indices``  -- a1 / O2-O3.  Frame set *I* (Alg. 1 l.3 P:362)
  by HF ``Qwen2VLVideoProcessor.sample_frames`` semantics (reading R1).
  Pinned: vs transformers on all configs + sweep (tests/test_oracle_pins.py).
* ``smart_resize``   -- a2 / O4 (reading R2).  Pinned: brute force vs transformers.
* ``grid_thw``       -- O5; closed form ceil(n/2)*H'/14*W'/14 (north star).
* ``check_rank_plans`` -- O6 / O12: invariants of a W-rank plan (P:339-340,
  method b; GOP indivisibility P:315/P:328).  Any valid plan gives the same
  concatenated tokens, so only validity is checked, plus
  ``brute_force_min_max_pairs`` for optimality on tiny inputs.
* ``preprocess``     -- O7..O11 via the plain C library ``liboracle.so``
  (fc_oracle.c): BT.601, Pillow bicubic, HF normalize, Qwen2-VL patch order;
  ``backend="torchvision"`` (R21): torch's uint8 antialiased bicubic and HF's
  fused normalisation, pinned against torch and Qwen2VLVideoProcessor.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from fractions import Fraction
from itertools import combinations

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

CLIP_MEAN = (0.48145466, 0.4578275, 0.40821073)
CLIP_STD = (0.26862954, 0.26130258, 0.27577711)
PATCH, TPS, MERGE = 14, 2, 2
COLS = 3 * TPS * PATCH * PATCH  # 1176


# ------------------------------------------------------------------ build --
def build(force: bool = False) -> str:
    """Compile fc_oracle.c -> liboracle.so (plain gcc, no FMA contraction)."""
    src = os.path.join(HERE, "fc_oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                               "-pthread", "-o", LIB_PATH, src, "-lm"])
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        u8p = ctypes.POINTER(ctypes.c_uint8)
        L.oracle_bt601_pixel.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, u8p]
        L.oracle_nv12_to_rgb.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                         ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
        L.oracle_resize_coeffs.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
        L.oracle_resize_coeffs.restype = ctypes.c_int
        L.oracle_resize_bicubic.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                            ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
        L.oracle_resize_bicubic.restype = ctypes.c_int
        L.oracle_normalize.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_double, ctypes.c_int]
        L.oracle_normalize.restype = ctypes.c_float
        L.oracle_tokens.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double, ctypes.c_int, ctypes.c_void_p]
        L.oracle_preprocess.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.oracle_yuv_coeffs.argtypes = [ctypes.c_int, ctypes.c_void_p]
        L.oracle_codes.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
        L.oracle_yuv_pixel.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, u8p]
        L.oracle_yuv_table.argtypes = [ctypes.c_int, ctypes.c_void_p]
        L.oracle_preprocess.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# --------------------------------------------------------------- a1 sampling --
def sample_indices(num_frames_total: int, fps_src: Fraction | float, sample_fps: float | None = 2.0,
                   min_frames: int = 4, max_frames: int = 768, tps: int = TPS,
                   num_frames: int | None = None, mode: str = "fps_stride",
                   explicit: list[int] | None = None) -> list[int]:
    """Frame set I -- reading R1 (HF sample_frames, transformers
    models/qwen2_vl/video_processing_qwen2_vl.py:155-190):

        maxf = floor(min(max_frames, N)/tps)*tps
        n    = floor(min(max(N/fps_src*fps, min_frames), maxf, N)/tps)*tps   (f64)
        idx_i = floor(i*N/n)                                               (exact ints)

    ``num_frames`` given: n = round(num_frames/tps)*tps (Python round).
    ``mode='linspace'``: idx_i = round_half_even(i*(N-1)/(n-1)) (qwen-vl-utils).
    ``mode='explicit'``: the strictly increasing list as given.
    Raises ValueError for an empty selection or n > N (HF's ValueError).
    """
    N = int(num_frames_total)
    if mode == "explicit":
        idx = [int(i) for i in (explicit or [])]
        if not idx or any(b <= a for a, b in zip(idx, idx[1:])) or idx[0] < 0 or idx[-1] >= N:
            raise ValueError("invalid explicit selection")
        return idx
    if num_frames is not None:
        n = round(num_frames / tps) * tps
    else:
        fps_src_f = float(fps_src)
        maxf = math.floor(min(max_frames, N) / tps) * tps
        x = N / fps_src_f * sample_fps
        x = min(max(x, min_frames), maxf, N)
        n = math.floor(x / tps) * tps
    if n <= 0 or n > N:
        raise ValueError(f"empty selection (n={n}, N={N})")
    if mode == "linspace":
        if n == 1:
            return [0]
        return [round(Fraction(i * (N - 1), n - 1)) for i in range(n)]
    return [(i * N) // n for i in range(n)]


# ------------------------------------------------------------- a2 resize --
def video_max_pixels(min_pixels: int, max_pixels: float, total_pixels: float, n: int, tps: int = TPS) -> float:
    """Reading R2, optional total budget (qwen-vl-utils'
    fetch_video): the per-frame budget becomes
        max(min(max_pixels, total_pixels / n * tps), int(min_pixels * 1.05))
    kept as f64 (int() truncates; min_pixels * 1.05 > 0)."""
    return max(min(max_pixels, total_pixels / n * tps), int(min_pixels * 1.05))


def smart_resize(height: int, width: int, factor: int = 28, min_pixels: int = 128 * 28 * 28,
                 max_pixels: float = 768 * 28 * 28, total_pixels: float = 0.0, n: int = 0) -> tuple[int, int]:
    """Reading R2: HF smart_resize (transformers models/qwen2_vl/
    image_processing_qwen2_vl.py:62-88), Python round-half-even, f64.
    ``total_pixels > 0`` (with the sampled frame count ``n``) first lowers the
    per-frame budget by :func:`video_max_pixels`."""
    if total_pixels > 0:
        max_pixels = video_max_pixels(min_pixels, max_pixels, total_pixels, n)
    if max(height, width) / min(height, width) > 200:
        raise ValueError("aspect ratio > 200")
    h_bar = round(height / factor) * factor
    w_bar = round(width / factor) * factor
    if h_bar * w_bar > max_pixels:
        beta = math.sqrt((height * width) / max_pixels)
        h_bar = max(factor, math.floor(height / beta / factor) * factor)
        w_bar = max(factor, math.floor(width / beta / factor) * factor)
    elif h_bar * w_bar < min_pixels:
        beta = math.sqrt(min_pixels / (height * width))
        h_bar = math.ceil(height * beta / factor) * factor
        w_bar = math.ceil(width * beta / factor) * factor
    return h_bar, w_bar


def grid_thw(n: int, h2: int, w2: int) -> tuple[int, int, int]:
    """O5: (ceil(n/T), H'/14, W'/14); token rows = product (north star)."""
    return ((n + TPS - 1) // TPS, h2 // PATCH, w2 // PATCH)


# --------------------------------------------------------- O6 plan checks --
def gop_of(frame: int, gop_start: list[int]) -> int:
    g = 0
    while g + 1 < len(gop_start) and gop_start[g + 1] <= frame:
        g += 1
    return g


def check_rank_plans(gop_start: list[int], num_frames: int, sampled: list[int], world: int,
                     ranks: list[dict], gh: int, gw: int) -> None:
    """Assert the invariants of a W-rank plan (P:339-340 method b, P:315/328
    GOP indivisibility).  ``ranks[r]`` has keys gop_begin,
    gop_end, tail_gop, tail_frame, sampled_begin, sampled_count, pad_frames,
    row_begin, row_end.  Raises AssertionError on the first violation."""
    n = len(sampled)
    G = len(gop_start)
    assert len(ranks) == world
    pos = 0
    row = 0
    nonempty = [r for r in range(world) if ranks[r]["sampled_count"] + ranks[r]["pad_frames"] > 0]
    # empty ranks are compacted to the end ("merge it away")
    assert nonempty == list(range(len(nonempty))), "empty ranks must be at the end"
    last = nonempty[-1] if nonempty else -1
    for r in range(world):
        rp = ranks[r]
        cnt = rp["sampled_count"]
        # contiguous cover of the sampled sequence, in time order
        assert rp["sampled_begin"] == pos, f"rank {r} begins at {rp['sampled_begin']}, expected {pos}"
        pos += cnt
        if r != last:
            assert rp["pad_frames"] == 0, "padding only on the last non-empty rank (P:339)"
        tot = cnt + rp["pad_frames"]
        if r != last and tot:
            assert tot % TPS == 0, f"rank {r} count {tot} not divisible by T (P:340)"
        # rows
        assert rp["row_begin"] == row
        assert rp["row_end"] - rp["row_begin"] == (tot // TPS) * gh * gw
        row = rp["row_end"]
        if cnt == 0:
            continue
        frames = sampled[rp["sampled_begin"]:rp["sampled_begin"] + cnt]
        g0, g1 = rp["gop_begin"], rp["gop_end"]
        assert 0 <= g0 < g1 <= G
        tail = rp["tail_frame"]
        body = [f for f in frames if f != tail] if tail >= 0 else frames
        if tail >= 0:
            assert frames[-1] == tail and rp["tail_gop"] == gop_of(tail, gop_start)
            assert rp["tail_gop"] >= g1, "tail frame lies beyond the owned GOP range"
        # owned GOP ranges are disjoint and increasing; they hold the body
        # frames (GOPs indivisible)
        if r > 0 and ranks[r - 1]["sampled_count"]:
            assert ranks[r - 1]["gop_end"] <= g0, "GOP ranges overlap"
        for f in body:
            assert g0 <= gop_of(f, gop_start) < g1, f"frame {f} outside rank {r} GOPs [{g0},{g1})"
    assert pos == n, "every sampled frame exactly once"
    # padding: only to make the grand total divisible by T
    total = n + sum(rp["pad_frames"] for rp in ranks)
    assert total % TPS == 0 and sum(rp["pad_frames"] for rp in ranks) == (-n) % TPS
    assert row == ((n + TPS - 1) // TPS) * gh * gw


def method_b_pairs(seg_counts: list[int]) -> list[int]:
    """Method b (Fig. 8b), reading R8: rank r's frames are the sampled
    positions [start_r, end_r) with start_0 = 0, start_r = end_{r-1},
    end_r = max(a_{r+1}, start_r) where a are the segment boundaries; if
    end_r - start_r is odd and frames remain, rank r also takes the next
    sampled frame in time (end_r += 1).  The last rank ends at n and pads
    with the last frame.  Returns the temporal pairs per rank."""
    bounds = [0]
    for c in seg_counts:
        bounds.append(bounds[-1] + c)
    n = bounds[-1]
    k = len(seg_counts)
    pairs = []
    start = 0
    for r in range(k):
        if r == k - 1:
            end = n
        else:
            end = max(bounds[r + 1], start)
            if (end - start) % TPS and end < n:
                end += TPS - (end - start) % TPS
                end = min(end, n)
        pairs.append((end - start + TPS - 1) // TPS)
        start = end
    return pairs


def brute_force_min_max_pairs(per_gop_counts: list[int], world: int) -> int:
    """Minimum over every contiguous GOP partition into <= W ranks of the
    max per-rank temporal pairs after method-b alignment (tiny inputs)."""
    G = len(per_gop_counts)
    best = None
    for k in range(1, min(world, G) + 1):
        for cuts in combinations(range(1, G), k - 1):
            b = (0,) + cuts + (G,)
            segs = [sum(per_gop_counts[b[i]:b[i + 1]]) for i in range(k)]
            m = max(method_b_pairs(segs))
            best = m if best is None else min(best, m)
    return best


# ------------------------------------------------------ O7..O11 pixels --
def nv12_to_rgb(y: np.ndarray, uv: np.ndarray, width: int, height: int) -> np.ndarray:
    """O7 on one frame; y: [H, pitch] u8, uv: [H/2, pitch] u8."""
    y = np.ascontiguousarray(y, dtype=np.uint8)
    uv = np.ascontiguousarray(uv, dtype=np.uint8)
    out = np.empty((height, width, 3), np.uint8)
    lib().oracle_nv12_to_rgb(_ptr(y), y.shape[1], _ptr(uv), uv.shape[1], width, height, _ptr(out))
    return out


def bt601_pixel(Y: int, U: int, V: int) -> tuple[int, int, int]:
    o = (ctypes.c_uint8 * 3)()
    lib().oracle_bt601_pixel(Y, U, V, o)
    return tuple(o)


MATRICES = {"bt601": 0, "bt709": 1, "bt601_full": 2, "bt709_full": 3}


def yuv_coeffs(matrix: str) -> tuple[int, ...]:
    """R15: (cY, y0, cRV, cGU, cGV, cBU) of a colour matrix."""
    k = np.empty(6, np.int32)
    lib().oracle_yuv_coeffs(MATRICES[matrix], _ptr(k))
    return tuple(int(x) for x in k)


def yuv_table(matrix: str) -> np.ndarray:
    """Every (Y, U, V) through oracle_yuv_pixel: [256, 256, 256, 3] u8."""
    out = np.empty((256, 256, 256, 3), np.uint8)
    lib().oracle_yuv_table(MATRICES[matrix], _ptr(out))
    return out


def to_bf16(x: np.ndarray) -> np.ndarray:
    """R16: fp32 -> bfloat16 bits, round to nearest, ties to even (finite
    inputs): keep the top 16 bits of b + 0x7FFF + (bit 16 of b)."""
    b = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    return ((b + 0x7FFF + ((b >> 16) & 1)) >> 16).astype(np.uint16)


BACKENDS = {"pil": 0, "torchvision": 1}  # reading R21 (fc_oracle.c make_coeffs / oracle_normalize)


def resize_bicubic(rgb: np.ndarray, w2: int, h2: int, backend: str = "pil") -> np.ndarray:
    """O8 bicubic on an [H, W, 3] u8 image: Pillow-exact ("pil") or torch's
    uint8 antialiased bicubic ("torchvision", R21)."""
    rgb = np.ascontiguousarray(rgb, dtype=np.uint8)
    h, w = rgb.shape[:2]
    out = np.empty((h2, w2, 3), np.uint8)
    if lib().oracle_resize_bicubic(_ptr(rgb), w, h, w2, h2, BACKENDS[backend], _ptr(out)) != 0:
        raise MemoryError
    return out


def resize_coeffs(n_in: int, n_out: int, backend: str = "pil", with_precision: bool = False):
    b = BACKENDS[backend]
    ks = lib().oracle_resize_coeffs(n_in, n_out, b, None, None, None, 0, None)
    xmin = np.empty(n_out, np.int32)
    cnt = np.empty(n_out, np.int32)
    iw = np.empty(n_out * ks, np.int32)
    prec = ctypes.c_int(0)
    lib().oracle_resize_coeffs(n_in, n_out, b, _ptr(xmin), _ptr(cnt), _ptr(iw), ks, ctypes.byref(prec))
    if with_precision:
        return xmin, cnt, iw.reshape(n_out, ks), prec.value
    return xmin, cnt, iw.reshape(n_out, ks)


def normalize_value(v: int, ch: int, mean=CLIP_MEAN, std=CLIP_STD, rescale: float = 1 / 255,
                    backend: str = "pil") -> np.float32:
    m = np.array(mean, np.float32)
    s = np.array(std, np.float32)
    return np.float32(lib().oracle_normalize(v, ch, _ptr(m), _ptr(s), rescale, BACKENDS[backend]))


def tokens_from_resized(rs: np.ndarray, mean=CLIP_MEAN, std=CLIP_STD, rescale: float = 1 / 255,
                        backend: str = "pil") -> np.ndarray:
    """O10-O11 on [n, H', W', 3] u8 resized frames."""
    rs = np.ascontiguousarray(rs, dtype=np.uint8)
    n, h2, w2 = rs.shape[:3]
    gt, gh, gw = grid_thw(n, h2, w2)
    out = np.empty((gt * gh * gw, COLS), np.float32)
    m = np.array(mean, np.float32)
    s = np.array(std, np.float32)
    lib().oracle_tokens(_ptr(rs), n, w2, h2, _ptr(m), _ptr(s), rescale, BACKENDS[backend], _ptr(out))
    return out


def codes_from_resized(rs: np.ndarray) -> np.ndarray:
    """NEXT-1 exchange format: the R6 layout of the resized u8 values."""
    rs = np.ascontiguousarray(rs, dtype=np.uint8)
    n, h2, w2 = rs.shape[:3]
    gt, gh, gw = grid_thw(n, h2, w2)
    out = np.empty((gt * gh * gw, COLS), np.uint8)
    lib().oracle_codes(_ptr(rs), n, w2, h2, _ptr(out))
    return out


def i420_chroma_to_nv12(u: np.ndarray, v: np.ndarray, width: int) -> np.ndarray:
    """Planar U, V rows (I420) -> the interleaved U,V rows of NV12 holding the
    same samples: uv[r][2i] = U[r][i], uv[r][2i+1] = V[r][i] (the two layouts
    are the same 4:2:0 samples; north star "NV12/YUV420 surfaces")."""
    cw = width // 2
    uv = np.empty((u.shape[0], width), np.uint8)
    uv[:, 0::2] = u[:, :cw]
    uv[:, 1::2] = v[:, :cw]
    return uv


def preprocess_i420(frames, width: int, height: int, w2: int, h2: int, **kw):
    """O7..O11 on I420 frames (y, u, v): chroma interleaved, then `preprocess`."""
    return preprocess([(y, i420_chroma_to_nv12(u, v, width)) for y, u, v in frames], width, height, w2, h2, **kw)


def preprocess(frames: list[tuple[np.ndarray, np.ndarray]], width: int, height: int, w2: int, h2: int,
               mean=CLIP_MEAN, std=CLIP_STD, rescale: float = 1 / 255, want_rgb: bool = False,
               nthreads: int = 1, matrix: str = "bt601", backend: str = "pil"):
    """O7..O11 end to end on the *sampled* frames (in order), each a pair
    (y [H, pitch_y] u8, uv [H/2, pitch_uv] u8).  Returns tokens
    [ceil(n/2)*gh*gw, 1176] f32 (and the RGB dumps if ``want_rgb``)."""
    n = len(frames)
    ys = [np.ascontiguousarray(f[0], dtype=np.uint8) for f in frames]
    uvs = [np.ascontiguousarray(f[1], dtype=np.uint8) for f in frames]
    yp = (ctypes.c_void_p * n)(*[y.ctypes.data for y in ys])
    uvp = (ctypes.c_void_p * n)(*[u.ctypes.data for u in uvs])
    py = np.array([y.shape[1] for y in ys], np.int64)
    puv = np.array([u.shape[1] for u in uvs], np.int64)
    gt, gh, gw = grid_thw(n, h2, w2)
    tokens = np.empty((gt * gh * gw, COLS), np.float32)
    rgb_src = np.empty((n, height, width, 3), np.uint8) if want_rgb else None
    rgb_rs = np.empty((n, h2, w2, 3), np.uint8)
    m = np.array(mean, np.float32)
    s = np.array(std, np.float32)
    st = lib().oracle_preprocess(yp, uvp, _ptr(py), _ptr(puv), n, width, height, w2, h2, _ptr(m), _ptr(s),
                                 rescale, _ptr(tokens), _ptr(rgb_src) if want_rgb else None, _ptr(rgb_rs),
                                 nthreads, MATRICES[matrix], BACKENDS[backend])
    if st != 0:
        raise RuntimeError("oracle_preprocess failed")
    if want_rgb:
        return tokens, rgb_src, rgb_rs
    return tokens
