"""Host planner (fc_plan, through the C ABI) vs the oracle -- CPU only.

Covers rows a1-a4 and b of SURVEY §8: sampling indices and grid_thw
bit-exact against the oracle, the GOP partition's invariants (P:339-340,
method b), optimality of the DP against brute force
on tiny inputs, structured errors, and that libfc.so
loads and exports every symbol include/fc.h declares.
"""
import ctypes
import os
import random
import re

import numpy as np

import pytest

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def plan_of(fc, W, H, N, gops, fps=(30, 1), **cfg):
    return fc.Plan(fc.VideoMeta(W, H, N, fps, gops), fc.ModelCfg(**cfg))


def test_abi_exports_every_declared_symbol(fc):
    hdr = open(os.path.join(ROOT, "include", "fc.h")).read()
    names = set(re.findall(r"\b(fc_[a-z0-9_]+)\s*\(", hdr))
    assert len(names) >= 15
    lib = ctypes.CDLL(fc._native.LIB_PATH)
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing
    assert fc.lib().fc_abi_version() == fc._native.ABI_VERSION
    m = re.search(r"#define FC_ABI_VERSION (\d+)", hdr)
    assert m and int(m.group(1)) == fc._native.ABI_VERSION


@pytest.mark.parametrize("name", sorted(synth.CONFIGS))
def test_config_plans_match_oracle(fc, oracle, name):
    wl = synth.CONFIGS[name]
    for world in (1, 2, 4, 8):
        p = plan_of(fc, wl.width, wl.height, wl.num_frames, wl.gop_start, wl.fps, world_size=world,
                    sample_fps=wl.sample_fps)
        idx = oracle.sample_indices(wl.num_frames, wl.fps[0] / wl.fps[1], wl.sample_fps)
        assert p.sampled_indices == idx
        h2, w2 = oracle.smart_resize(wl.height, wl.width)
        assert p.resized == (h2, w2)
        assert p.grid_thw == oracle.grid_thw(len(idx), h2, w2)
        gt, gh, gw = p.grid_thw
        oracle.check_rank_plans(wl.gop_start, wl.num_frames, idx, world, p.ranks(), gh, gw)


def test_paper_scale_bottlenecks(fc):
    """Per-rank pairs at W=8: c2 8, c3 38, c4 4."""
    for name, want in (("c2", 8), ("c3", 38), ("c4", 4)):
        wl = synth.CONFIGS[name]
        p = plan_of(fc, wl.width, wl.height, wl.num_frames, wl.gop_start, wl.fps, world_size=8,
                    sample_fps=wl.sample_fps)
        pairs = [(r["sampled_count"] + r["pad_frames"]) // 2 for r in p.ranks()]
        assert max(pairs) == want, pairs


def test_single_gop_stays_on_encoder_rank(fc):
    # a GOP is indivisible; one GOP -> one rank (the encoder rank 0)
    wl = synth.CONFIGS["c1"]
    p = plan_of(fc, wl.width, wl.height, wl.num_frames, wl.gop_start, world_size=8)
    rs = p.ranks()
    assert rs[0]["sampled_count"] == 8 and all(r["sampled_count"] == 0 for r in rs[1:])
    assert p.ranks_used == 1


def _random_video(rng):
    G = rng.randint(1, 12)
    sizes = [rng.randint(1, 9) for _ in range(G)]
    N = sum(sizes)
    starts = [sum(sizes[:i]) for i in range(G)]
    return N, starts


def test_random_plans_invariants_and_optimality(fc, oracle):
    """1000 random (meta, selection, W): invariants hold; the max
    per-rank pairs equals the brute-force optimum."""
    rng = random.Random(1234)
    checked = 0
    for _ in range(1000):
        N, starts = _random_video(rng)
        k = rng.randint(1, N)
        explicit = sorted(rng.sample(range(N), k))
        world = rng.randint(1, 5)
        p = plan_of(fc, 64, 48, N, starts, world_size=world, sampling="explicit", explicit_indices=explicit)
        assert p.sampled_indices == explicit
        gt, gh, gw = p.grid_thw
        oracle.check_rank_plans(starts, N, explicit, world, p.ranks(), gh, gw)
        if len(starts) <= 8:
            per_gop = [sum(1 for f in explicit if oracle.gop_of(f, starts) == g) for g in range(len(starts))]
            best = oracle.brute_force_min_max_pairs(per_gop, world)
            got = max((r["sampled_count"] + r["pad_frames"] + 1) // 2 for r in p.ranks())
            assert got == best, (per_gop, world, got, best)
            checked += 1
    assert checked > 300


def test_monotone_in_world_size(fc):
    # more ranks never increase the bottleneck
    wl = synth.CONFIGS["c3"]
    prev = None
    for world in range(1, 9):
        p = plan_of(fc, wl.width, wl.height, wl.num_frames, wl.gop_start, world_size=world, sample_fps=1.0)
        m = max((r["sampled_count"] + r["pad_frames"]) // 2 for r in p.ranks())
        assert prev is None or m <= prev
        prev = m


def test_method_b_moves_frames_up_never_down(fc, oracle):
    # Fig. 8 / P:340: odd ranks take the next frame; only the last rank pads
    p = plan_of(fc, 64, 48, 30, [0, 10, 20], world_size=3, sampling="explicit",
                explicit_indices=[0, 3, 6, 10, 13, 16, 20, 23, 26])
    rs = p.ranks()
    assert [r["sampled_count"] for r in rs] == [4, 2, 3] or sum(r["pad_frames"] for r in rs) == 1
    assert all(r["pad_frames"] == 0 for r in rs[:-1] if r["sampled_count"])
    assert sum(r["sampled_count"] for r in rs) == 9
    for r in rs:
        if r["tail_frame"] >= 0:
            assert r["tail_gop"] >= r["gop_end"]


def test_est_decode_frames(fc):
    # decode from the keyframe through the last target of each GOP
    p = plan_of(fc, 64, 48, 30, [0, 10, 20], world_size=1, sampling="explicit", explicit_indices=[2, 5, 12, 25])
    assert p.rank(0)["est_decode_frames"] == (5 + 1) + (2 + 1) + (5 + 1)


def test_determinism(fc):
    wl = synth.CONFIGS["c2"]
    a = plan_of(fc, wl.width, wl.height, wl.num_frames, wl.gop_start, world_size=8)
    b = plan_of(fc, wl.width, wl.height, wl.num_frames, wl.gop_start, world_size=8)
    assert a.ranks() == b.ranks() and a.sampled_indices == b.sampled_indices


def test_encoder_rank_takes_a_full_share(fc):
    wl = synth.CONFIGS["c2"]
    p = plan_of(fc, wl.width, wl.height, wl.num_frames, wl.gop_start, world_size=8)
    pairs = [(r["sampled_count"] + r["pad_frames"]) // 2 for r in p.ranks()]
    assert pairs[0] == max(pairs)  # tie-break: maximise the encoder's share (fewer gather bytes)


def test_fixed_resize_paper_224(fc):
    # the serving evaluation resizes everything to 224x224
    p = plan_of(fc, 1920, 1080, 1800, list(range(0, 1800, 30)), resized_height=224, resized_width=224)
    assert p.resized == (224, 224) and p.grid_thw == (60, 16, 16)
    assert p.token_rows // p.grid_thw[0] == 256  # 128 patch rows per frame (R14)


@pytest.mark.parametrize("kwargs,code", [
    (dict(W=63, H=48), "FC_ERR_UNSUPPORTED"),           # odd width (NV12)
    (dict(W=64, H=48, N=1, gops=[0]), "FC_ERR_EMPTY_SELECTION"),  # n = 0
    (dict(W=4000, H=4, N=100), "FC_ERR_ASPECT_RATIO"),  # > 200:1
    (dict(gops=[0, 5, 5]), "FC_ERR_INVALID_ARG"),       # not strictly increasing
    (dict(gops=[1, 5]), "FC_ERR_INVALID_ARG"),          # first GOP must start at 0
    (dict(gops=[0, 500]), "FC_ERR_INVALID_ARG"),        # GOP start past the end
    (dict(cfg=dict(world_size=2, encoder_rank=2)), "FC_ERR_RANK"),
    (dict(cfg=dict(resized_height=100, resized_width=224)), "FC_ERR_INVALID_ARG"),
    (dict(cfg=dict(sampling="explicit", explicit_indices=[3, 2])), "FC_ERR_INVALID_ARG"),
])
def test_structured_errors(fc, kwargs, code):
    W, H, N = kwargs.get("W", 64), kwargs.get("H", 48), kwargs.get("N", 100)
    gops = kwargs.get("gops", [0, 50])
    with pytest.raises(fc.FcError) as e:
        plan_of(fc, W, H, N, gops, **kwargs.get("cfg", {}))
    assert e.value.name == code


def test_rank_out_of_range(fc):
    p = plan_of(fc, 64, 48, 100, [0, 50], world_size=2)
    with pytest.raises(fc.FcError) as e:
        p.rank(2)
    assert e.value.name == "FC_ERR_RANK"


def test_no_cpu_fallback(fc):
    """fc_preprocess must fail loudly (not compute on the CPU) without an sm_100 device."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    p = plan_of(fc, 64, 48, 100, [0, 50], sampling="explicit", explicit_indices=[0, 10])
    buf = (ctypes.c_uint8 * (48 * 64 * 2 + 64))()
    base = (ctypes.addressof(buf) + 15) & ~15
    surf = fc.SurfaceTable(100)
    for i in (0, 10):
        surf.arr[i] = fc._native.Nv12SurfaceC(base, base + 48 * 64, 64, 64)
    out = (ctypes.c_float * (p.token_rows * 1176))()
    st = fc.lib().fc_preprocess(p.handle, 0, surf.arr, 100, ctypes.cast(out, ctypes.c_void_p), None, None)
    assert fc._native.STATUS[st] == "FC_ERR_CUDA"
    assert b"sm_100" in fc.lib().fc_last_error() or b"cuda" in fc.lib().fc_last_error().lower()


def test_no_cpu_fallback_submit_and_tc(fc, monkeypatch):
    """fc_submit and the tcgen05 route (FC_TC=1) fail loudly too without an
    sm_100 device: no plan is returned, nothing computes on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    buf = (ctypes.c_uint8 * (48 * 64 * 2 + 64))()
    base = (ctypes.addressof(buf) + 15) & ~15
    surf = fc.SurfaceTable(100)
    for i in (0, 10):
        surf.arr[i] = fc._native.Nv12SurfaceC(base, base + 48 * 64, 64, 64)
    meta = fc.VideoMeta(64, 48, 100, (30, 1), [0, 50])
    cfg = fc.ModelCfg(sampling="explicit", explicit_indices=[0, 10])
    m, _km = meta.to_c()
    c, _kc = cfg.to_c()
    out = (ctypes.c_float * (28 * 1176 * 4))()
    h = ctypes.c_void_p()
    for tc in ("0", "1"):
        monkeypatch.setenv("FC_TC", tc)
        st = fc.lib().fc_submit(ctypes.byref(m), ctypes.byref(c), 0, surf.arr, 100, ctypes.cast(out, ctypes.c_void_p),
                                None, ctypes.byref(h))
        assert fc._native.STATUS[st] == "FC_ERR_CUDA" and not h.value
        assert fc.lib().fc_last_kernel() == 0  # no launch happened on this thread


def test_ipc_and_submit_argument_errors(fc):
    """Host-side validation of the round-2 entry points (no CUDA call needed)."""
    h = (ctypes.c_uint8 * 64)()
    assert fc._native.STATUS[fc.lib().fc_ipc_export(None, h)] == "FC_ERR_INVALID_ARG"
    assert fc._native.STATUS[fc.lib().fc_ipc_import(None, None)] == "FC_ERR_INVALID_ARG"
    assert fc._native.STATUS[fc.lib().fc_ipc_close(None)] == "FC_ERR_INVALID_ARG"
    off = ctypes.c_int64()
    assert fc._native.STATUS[fc.lib().fc_ipc_export_range(None, h, ctypes.byref(off))] == "FC_ERR_INVALID_ARG"
    assert fc._native.STATUS[fc.lib().fc_submit(None, None, 0, None, 0, None, None, None)] == "FC_ERR_INVALID_ARG"
    n = ctypes.c_int32()
    assert fc._native.STATUS[fc.lib().fc_exchange_schedule(None, 0, 0, None, 0, ctypes.byref(n))] == "FC_ERR_INVALID_ARG"


def test_missing_surface_reported(fc):
    p = plan_of(fc, 64, 48, 100, [0, 50], sampling="explicit", explicit_indices=[0, 10])
    surf = fc.SurfaceTable(100)  # all NULL
    out = (ctypes.c_float * (p.token_rows * 1176))()
    st = fc.lib().fc_preprocess(p.handle, 0, surf.arr, 100, ctypes.cast(out, ctypes.c_void_p), None, None)
    assert fc._native.STATUS[st] == "FC_ERR_MISSING_SURFACE"


@pytest.mark.parametrize("planes,status", [
    ("y u v", "FC_ERR_CUDA"),                  # valid I420 surfaces reach the device check (no GPU here)
    ("y u -", "FC_ERR_MISSING_SURFACE"),       # no V plane
    ("y u v+8", "FC_ERR_UNSUPPORTED"),         # V plane not 16-byte aligned
    ("y u v pitch16", "FC_ERR_UNSUPPORTED"),   # chroma pitch < width / 2
])
def test_i420_surface_validation(fc, planes, status):
    """I420 surfaces (ABI 3: U in `uv`, V in `v`, shared chroma pitch >= W/2)
    are validated before any device work."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    p = plan_of(fc, 64, 48, 100, [0, 50], sampling="explicit", explicit_indices=[0, 10], surface_format="i420")
    buf = (ctypes.c_uint8 * (48 * 64 * 3 + 256))()
    base = (ctypes.addressof(buf) + 15) & ~15
    ub, vb = base + 48 * 64, base + 48 * 64 + 24 * 64
    surf = fc.SurfaceTable(100)
    for i in (0, 10):
        v = None if planes.endswith("-") else vb + (8 if planes.endswith("v+8") else 0)
        surf.arr[i] = fc._native.Nv12SurfaceC(base, ub, 64, 16 if planes.endswith("pitch16") else 32, v)
    out = (ctypes.c_float * (p.token_rows * 1176))()
    st = fc.lib().fc_preprocess(p.handle, 0, surf.arr, 100, ctypes.cast(out, ctypes.c_void_p), None, None)
    assert fc._native.STATUS[st] == status, fc.lib().fc_last_error()


@pytest.mark.parametrize("field,value", [("token_dtype", 3), ("color", 4), ("color", -1), ("surface_format", 2),
                                         ("backend", 2), ("backend", -1)])
def test_unknown_variant_enums_rejected(fc, field, value):
    """NEXT-4 variant enums are validated by fc_plan (S:34 structured errors)."""
    meta = fc.VideoMeta(64, 48, 100, (30, 1), [0, 50])
    m, _k1 = meta.to_c()
    c, _k2 = fc.ModelCfg().to_c()
    setattr(c, field, value)
    h = ctypes.c_void_p()
    st = fc.lib().fc_plan(ctypes.byref(m), ctypes.byref(c), ctypes.byref(h))
    assert fc._native.STATUS[st] == "FC_ERR_UNSUPPORTED"


def test_model_cfg_struct_matches_abi(fc):
    """The ctypes mirror of fc_model_cfg has the C layout: fc_model_cfg_default
    fills the trailing fields with their documented defaults."""
    c = fc._native.ModelCfgC()
    c.token_dtype, c.color, c.surface_format, c.backend = 9, 9, 9, 9
    fc.lib().fc_model_cfg_default(ctypes.byref(c))
    assert (c.token_dtype, c.color, c.surface_format, c.world_size, c.encoder_rank, c.backend) == (0, 0, 0, 1, 0, 0)
    assert abs(c.rescale_factor - 1 / 255) < 1e-15 and c.patch_size == 14


@pytest.mark.parametrize("kw,ok", [
    (dict(page_rows=48), False),                      # not a power of two
    (dict(first_offset=64), False),                   # outside [0, page_rows)
    (dict(page_ids=[0]), False),                      # one page cannot hold first_offset + rows
    (dict(page_ids=[0, 9]), False),                   # page id outside the 8-page pool
    (dict(page_ids=[], first_offset=0), False),
])
def test_paged_output_validation(fc, kw, ok):
    """NEXT-2 write_chunk preconditions (SPEC CapacityError / bad page ids) are
    rejected before any device work: FC_ERR_INVALID_ARG, nothing launched."""
    p = plan_of(fc, 64, 48, 100, [0, 50], sampling="explicit", explicit_indices=[0, 10, 20, 30])
    rows = p.token_rows
    buf = (ctypes.c_uint8 * (48 * 64 * 2 + 64))()
    base = (ctypes.addressof(buf) + 15) & ~15
    surf = fc.SurfaceTable(100)
    for i in (0, 10, 20, 30):
        surf.arr[i] = fc._native.Nv12SurfaceC(base, base + 48 * 64, 64, 64)
    args = dict(page_rows=64, page_ids=[3], first_offset=60)
    args.update(kw)
    ids = (ctypes.c_int32 * max(1, len(args["page_ids"])))(*args["page_ids"])
    d = fc._native.PagedTokensC(ctypes.c_void_p(base), 8, args["page_rows"], len(args["page_ids"]),
                                ctypes.cast(ids, ctypes.POINTER(ctypes.c_int32)), args["first_offset"])
    st = fc.lib().fc_preprocess_paged(p.handle, 0, surf.arr, 100, ctypes.byref(d), None, None)
    assert rows > 4 and fc._native.STATUS[st] == "FC_ERR_INVALID_ARG"


def test_graft_entry_build_runs():
    """The driver's build check: __graft_entry__.build() compiles (or finds
    current) libfc.so + the oracle and checks the ABI version."""
    import importlib
    import sys
    sys.path.insert(0, ROOT)
    ge = importlib.import_module("__graft_entry__")
    ge.build()


def test_bicubic_output_range_fits_extended_table():
    """The V pass indexes the normalisation table at floor(S / 2^22) without a
    clamp (fc_fused.cuh kLutLo = 48: entries for v in [-48, 303]).  That needs
    every reachable Pillow-bicubic output (R4: S = 2^21 + sum px*iw, px in
    [0, 255]) inside the table.  Checked on the oracle's own coefficients over
    up- and downscales (the product checks the same bound per plan at launch)."""
    import random

    from oracle import oracle

    rng = random.Random(7)
    pairs = [(1080, 560), (720, 560), (2160, 560), (480, 476), (240, 280), (1080, 224), (2160, 28),
             (7, 28), (28, 56), (100, 201), (13, 1000)]
    pairs += [(rng.randint(2, 4000), rng.randint(28, 2000)) for _ in range(200)]
    lo, hi = 0, 255
    for n_in, n_out in pairs:
        _, cnt, iw = oracle.resize_coeffs(n_in, n_out)
        pos = np.where(iw > 0, iw, 0).astype(np.int64).sum(axis=1)
        neg = np.where(iw < 0, iw, 0).astype(np.int64).sum(axis=1)
        lo = min(lo, int((((1 << 21) + 255 * neg) >> 22).min()))
        hi = max(hi, int((((1 << 21) + 255 * pos) >> 22).max()))
    assert -48 <= lo and hi <= 303, (lo, hi)
    # the negative lobes of the a = -0.5 kernel integrate to 1/12 and, sampled
    # at a 2x upscale's half-pixel phase, sum to 1/8 of the normalised weights:
    # about [-32, 287]; integer rounding of small filters adds a little (M: [-34, 289])
    assert lo >= -40 and hi <= 295, (lo, hi)


def test_colsplit_requires_world_dividing_1176(fc):
    """NEXT-1 column split: W must divide 1176 (C = 1176 / W columns per
    block); W = 5 is rejected before any device work."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    p = plan_of(fc, 64, 48, 100, [0, 20, 40, 60, 80], sampling="explicit",
                explicit_indices=[0, 1, 20, 21, 40, 41, 60, 61, 80, 81], world_size=5)
    buf = (ctypes.c_uint8 * (48 * 64 * 2 + 64))()
    base = (ctypes.addressof(buf) + 15) & ~15
    surf = fc.SurfaceTable(100)
    for i in p.sampled_indices:
        surf.arr[i] = fc._native.Nv12SurfaceC(base, base + 48 * 64, 64, 64)
    out = (ctypes.c_float * 1176)()
    st = fc.lib().fc_preprocess_colsplit(p.handle, 0, surf.arr, 100, ctypes.cast(out, ctypes.c_void_p), None, None)
    assert fc._native.STATUS[st] == "FC_ERR_UNSUPPORTED", fc.lib().fc_last_error()
    st = fc.lib().fc_scatter_columns(p.handle, 0, None, None, ctypes.cast(out, ctypes.c_void_p), None)
    assert fc._native.STATUS[st] == "FC_ERR_UNSUPPORTED"


# ------------------------------------------------ a1/a2 planner modes
@pytest.mark.parametrize("N,n_req", [(100, 5), (100, 7), (1800, 120), (18000, 600), (300, 21), (9, 8), (64, 64)])
def test_num_frames_mode_matches_oracle(fc, oracle, N, n_req):
    """a1 `num_frames` rule (n = round_half_even(num_frames/2)*2) through
    fc_plan == the oracle (pinned to HF in test_oracle_pins)."""
    p = plan_of(fc, 320, 240, N, [0], num_frames=n_req)
    assert p.sampled_indices == oracle.sample_indices(N, 30, None, num_frames=n_req)


@pytest.mark.parametrize("N,fps", [(1800, 2.0), (120, 2.0), (18000, 1.0), (301, 0.5), (17, 2.0), (900, 2.0)])
def test_linspace_mode_matches_oracle(fc, oracle, N, fps):
    """a1 LINSPACE (idx_i = round_half_even(i(N-1)/(n-1)), exact rational)
    through fc_plan == the oracle."""
    p = plan_of(fc, 320, 240, N, [0], sampling="linspace", sample_fps=fps)
    assert p.sampled_indices == oracle.sample_indices(N, 30, fps, mode="linspace")


@pytest.mark.parametrize("total", [90_316_800, 1000, 5e6, 3.3e7, 1e12])
@pytest.mark.parametrize("WH", [(1280, 720), (1920, 1080), (854, 480), (3840, 2160), (320, 240)])
def test_total_pixels_budget_matches_oracle(fc, oracle, total, WH):
    """a2 optional total_pixels budget (qwen-vl-utils) through fc_plan == the
    oracle's pinned video_max_pixels + smart_resize (c3 variant: 728x392)."""
    W, H = WH
    p = plan_of(fc, W, H, 1800, list(range(0, 1800, 30)), total_pixels=total, sample_fps=2.0)
    n = len(p.sampled_indices)
    assert p.resized == oracle.smart_resize(H, W, total_pixels=total, n=n)
    assert p.grid_thw == oracle.grid_thw(n, *p.resized)


def test_c3_total_pixels_variant(fc):
    wl = synth.CONFIGS["c3"]
    p = plan_of(fc, wl.width, wl.height, wl.num_frames, wl.gop_start, wl.fps, sample_fps=1.0,
                total_pixels=90_316_800)
    assert p.resized == (392, 728) and p.grid_thw == (300, 28, 52) and p.token_rows == 436_800


def test_fractional_fps_sweep_matches_oracle(fc, oracle):
    """Q20 through the product: rational source rates (29.97 = 30000/1001, ...)
    x sampling rates x lengths -- fc_plan's indices equal the oracle's (which
    is pinned to HF's sample_frames up to the documented arange-length quirk)."""
    from fractions import Fraction
    rates = [Fraction(24), Fraction(25), Fraction(30), Fraction(60), Fraction(30000, 1001), Fraction(24000, 1001),
             Fraction(60000, 1001)]
    cases = 0
    for N in list(range(2, 600, 11)) + [1453, 1800, 4000]:
        for r in rates:
            for fps in (0.5, 1.0, 2.0):
                try:
                    want = oracle.sample_indices(N, r, fps)
                except ValueError:
                    with pytest.raises(fc.FcError):
                        plan_of(fc, 64, 48, N, [0], fps=(r.numerator, r.denominator), sample_fps=fps)
                    continue
                p = plan_of(fc, 64, 48, N, [0], fps=(r.numerator, r.denominator), sample_fps=fps)
                assert p.sampled_indices == want, (N, r, fps)
                cases += 1
    assert cases > 1000


# ------------------------------------------------ a10 exchange schedule
def _run_schedules(fc, plan, kind, elem):
    """Execute every rank's fc_exchange_schedule on host byte buffers (what
    fc_gather / fc_scatter_columns hand to NCCL) and return the receive
    buffers.  Send buffers: gather -> each rank's row shard of a reference
    token array; colsplit -> each rank's [W][rows][C] column blocks."""
    W = plan.world_size
    rows = plan.token_rows
    rng = np.random.default_rng(rows + W)
    full = rng.integers(0, 256, size=(rows, 1176 * elem), dtype=np.uint8)
    rps = plan.ranks()
    C = 1176 // W
    send, recv = [], []
    for r, rp in enumerate(rps):
        mine = full[rp["row_begin"]:rp["row_end"]]
        if kind == "gather":
            send.append(mine.tobytes())
            recv.append(bytearray(rows * 1176 * elem) if r == plan.cfg.encoder_rank else bytearray(0))
        else:
            f32 = mine.view(np.float32)  # [rows_r][1176]
            blocks = np.stack([f32[:, j * C:(j + 1) * C] for j in range(W)]) if len(f32) else np.zeros((W, 0, C))
            send.append(np.ascontiguousarray(blocks, dtype=np.float32).tobytes())
            recv.append(bytearray(rows * C * 4))
    scheds = [fc.exchange_schedule(plan, r, kind) for r in range(W)]
    covered = [np.zeros(len(recv[r]), dtype=np.int32) for r in range(W)]
    for r, xs in enumerate(scheds):
        for x in xs:
            if x["dir"] == "local":
                assert x["peer"] == r
                recv[r][x["dst_offset"]:x["dst_offset"] + x["bytes"]] = \
                    send[r][x["src_offset"]:x["src_offset"] + x["bytes"]]
                covered[r][x["dst_offset"]:x["dst_offset"] + x["bytes"]] += 1
            elif x["dir"] == "send":
                p = x["peer"]
                match = [y for y in scheds[p] if y["dir"] == "recv" and y["peer"] == r]
                assert len(match) == 1 and match[0]["bytes"] == x["bytes"], (r, p)
                y = match[0]
                recv[p][y["dst_offset"]:y["dst_offset"] + y["bytes"]] = \
                    send[r][x["src_offset"]:x["src_offset"] + x["bytes"]]
                covered[p][y["dst_offset"]:y["dst_offset"] + y["bytes"]] += 1
            else:  # every receive has exactly one matching send
                assert sum(1 for y in scheds[x["peer"]] if y["dir"] == "send" and y["peer"] == r) == 1
            assert 0 <= x["src_offset"] and x["bytes"] > 0
    return full, recv, covered


@pytest.mark.parametrize("seed", range(40))
def test_exchange_schedules_assemble_the_single_gpu_tensor(fc, seed):
    """fc_gather's and fc_scatter_columns' transfer lists, executed on host
    buffers: the encoder's buffer equals the single-GPU token array (every
    byte written exactly once, nothing else); after the column split rank j
    holds columns [jC, (j+1)C) of every row.  Random GOP layouts, explicit
    selections with method-b tails and padding, idle ranks, encoder != 0."""
    rng = random.Random(seed)
    N, starts = _random_video(rng)
    W = rng.choice([1, 2, 3, 4, 6, 7, 8])
    k = rng.randint(1, N)
    expl = sorted(rng.sample(range(N), k))
    enc = rng.randrange(W)
    tok = rng.choice(["f32", "bf16", "u8"])
    p = plan_of(fc, 56, 56, N, starts, world_size=W, encoder_rank=enc, sampling="explicit", explicit_indices=expl,
                token_dtype=tok)
    elem = {"f32": 4, "bf16": 2, "u8": 1}[tok]
    full, recv, covered = _run_schedules(fc, p, "gather", elem)
    assert bytes(recv[enc]) == full.tobytes()
    assert (covered[enc] == 1).all()
    if 1176 % W == 0 and tok == "f32":
        full, recv, covered = _run_schedules(fc, p, "colsplit", 4)
        C = 1176 // W
        f32 = full.view(np.float32)
        for j in range(W):
            got = np.frombuffer(bytes(recv[j]), dtype=np.float32).reshape(p.token_rows, C)
            np.testing.assert_array_equal(got, f32[:, j * C:(j + 1) * C])
            assert (covered[j] == 1).all()


def test_exchange_schedule_config_sizes(fc):
    """SURVEY 8(e) exchange sizes: c2 at W=8 moves 704.5 MB of fp32 rows into
    the encoder (1/8 of the 812.9 MB stays local), 4x less as u8 codes."""
    wl = synth.CONFIGS["c2"]
    for tok, mb in (("f32", 704.5), ("u8", 176.1)):
        p = plan_of(fc, wl.width, wl.height, wl.num_frames, wl.gop_start, wl.fps, world_size=8, token_dtype=tok)
        into = sum(x["bytes"] for x in fc.exchange_schedule(p, 0, "gather") if x["dir"] == "recv")
        assert abs(into / 1e6 - mb) < 0.1, into


def test_exchange_schedule_errors(fc):
    p = plan_of(fc, 64, 48, 8, [0], world_size=5)
    with pytest.raises(fc.FcError) as e:
        fc.exchange_schedule(p, 5)
    assert e.value.name == "FC_ERR_RANK"
    with pytest.raises(fc.FcError) as e:  # 1176 % 5 != 0
        fc.exchange_schedule(p, 0, "colsplit")
    assert e.value.name == "FC_ERR_UNSUPPORTED"


# ------------------------------------------------ throughput mode placement
def test_assign_requests_lpt(fc):
    """fc_assign_requests: every request placed once; equal requests (config 5:
    64 clips of 10 pairs) split evenly; LPT within Graham's 4/3 bound of the
    brute-force optimum on small random instances."""
    import itertools
    assert sorted(collections_count(fc.assign_requests([10] * 64, 8)).values()) == [8] * 8
    assert fc.assign_requests([], 4) == []
    rng = random.Random(3)
    for _ in range(200):
        n, w = rng.randint(1, 7), rng.randint(1, 4)
        pairs = [rng.randint(0, 20) for _ in range(n)]
        got = fc.assign_requests(pairs, w)
        assert len(got) == n and all(0 <= r < w for r in got)
        loads = [sum(p for p, r in zip(pairs, got) if r == k) for k in range(w)]
        opt = min(max(sum(p for p, r in zip(pairs, a) if r == k) for k in range(w))
                  for a in itertools.product(range(w), repeat=n))
        assert max(loads) <= opt * 4 / 3 + 1e-9 or max(loads) == opt, (pairs, w, got, opt)
    with pytest.raises(fc.FcError):
        fc.assign_requests([1, -1], 2)


def collections_count(xs):
    import collections
    return collections.Counter(xs)


def test_backend_shares_the_plan(fc):
    """R21: the torchvision backend plans like the PIL one (sampling, sizes,
    rank split are shared; only the resize and normalise tables differ)."""
    for W, H in [(1920, 1080), (320, 240), (854, 480)]:
        a = plan_of(fc, W, H, 120, list(range(0, 120, 30)), world_size=3)
        b = plan_of(fc, W, H, 120, list(range(0, 120, 30)), world_size=3, backend="torchvision")
        assert a.resized == b.resized and a.grid_thw == b.grid_thw and a.sampled_indices == b.sampled_indices
        assert [a.rank(r) for r in range(3)] == [b.rank(r) for r in range(3)]


def test_jpeg_decoder_argument_errors(fc):
    """fc_jpeg_* argument checks happen before any nvJPEG / device call."""
    h = ctypes.c_void_p()
    assert fc._native.STATUS[fc.lib().fc_jpeg_decoder_create(7, ctypes.byref(h))] == "FC_ERR_INVALID_ARG"
    assert fc._native.STATUS[fc.lib().fc_jpeg_decoder_create(0, None)] == "FC_ERR_INVALID_ARG"
    w = ctypes.c_int32()
    assert fc._native.STATUS[fc.lib().fc_jpeg_info(None, b"x", 1, ctypes.byref(w), ctypes.byref(w), None)] == \
        "FC_ERR_INVALID_ARG"
    assert fc.lib().fc_jpeg_decoder_backend(None) == -1
