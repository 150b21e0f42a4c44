"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle.

Bar (BASELINE.json north star):
  * sampling indices, grid_thw, the BT.601 RGB intermediate and the resized
    RGB intermediate: bit-exact;
  * normalised fp32 tokens: |gpu - oracle| <= 1e-5 * max(|oracle|, 1) per
    element (reading R7; bit-exact expected, and the count is reported).
Two fused kernels serve these requests: the mma.sync kernel (the default) and
the tcgen05 kernel (FC_TC=1: NV12 / fp32 wherever its shared-memory plan
fits) -- the `kernel` fixture runs a test through each.  Small cases are compared element by element on the whole
output, through both the production instance (fc_preprocess) and the debug
instance that also dumps the integer intermediates; the full BASELINE configs
run in the bench's launch configuration (one launch per rank, all frames) and
are compared element by element on the WHOLE token tensor against the
threaded oracle, in chunks of pairs.
"""
import os
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


def tol_check(got, ref, what=""):
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    tol = 1e-5 * np.maximum(np.abs(ref), 1.0)
    bad = np.abs(got - ref) > tol
    nbad = int(bad.sum())
    if nbad:
        i = np.argwhere(bad)[0]
        raise AssertionError(f"{what}: {nbad} elements out of tolerance, first at {tuple(i)}: "
                             f"gpu {got[tuple(i)]!r} oracle {ref[tuple(i)]!r}")
    return int((got.view(np.uint32) == ref.view(np.uint32)).sum())


def make_plan(fc, W, H, N, gops, world=1, **cfg):
    meta = fc.VideoMeta(W, H, N, (30, 1), gops)
    return fc.Plan(meta, fc.ModelCfg(world_size=world, **cfg))


def run_case(fc, oracle, cuda, W, H, N, gops, kind="natural", seed=7, world=1, check_rgb=True, **cfg):
    plan = make_plan(fc, W, H, N, gops, world, **cfg)
    idx = plan.sampled_indices
    pitch = synth.pitch_for(W)
    host = {i: synth.frame_nv12(W, H, i, kind, seed, pitch) for i in idx}
    dev = synth.to_device(host)
    surf = fc.SurfaceTable.from_tensors(dev, N)
    h2, w2 = plan.resized
    ref_tok, ref_src, ref_rs = oracle.preprocess([host[i] for i in idx], W, H, w2, h2, want_rgb=True,
                                                 matrix=cfg.get("color", "bt601"), backend=cfg.get("backend", "pil"))
    parts = []
    for r in range(world):
        rp = plan.rank(r)
        if rp["row_end"] == rp["row_begin"]:
            continue
        tok, src, rs = fc.preprocess_debug(plan, r, surf)
        cuda.cuda.synchronize()
        parts.append(tok.cpu().numpy())
        if check_rgb:
            fr = list(range(rp["sampled_begin"], rp["sampled_begin"] + rp["sampled_count"]))
            fr += [fr[-1]] * rp["pad_frames"]
            np.testing.assert_array_equal(src.cpu().numpy(), ref_src[fr], err_msg=f"rgb_src rank {r}")
            np.testing.assert_array_equal(rs.cpu().numpy(), ref_rs[fr], err_msg=f"rgb_resized rank {r}")
    got = np.concatenate(parts, axis=0)
    exact = tol_check(got, ref_tok, f"{W}x{H}->{w2}x{h2} {kind} W={world}")
    # the production instance (no dumps) on the same inputs, every rank
    prod = [fc.preprocess(plan, r, surf) for r in range(world) if plan.rank(r)["row_end"] > plan.rank(r)["row_begin"]]
    cuda.cuda.synchronize()
    got_p = np.concatenate([t.cpu().numpy() for t in prod], axis=0)
    assert tol_check(got_p, ref_tok, f"production {W}x{H}->{w2}x{h2} {kind} W={world}") == exact
    return plan, exact, got.size


@pytest.mark.parametrize("kind", ["natural", "uniform", "edges"])
def test_c1_shape_all_kinds(fc, oracle, cuda, kernel, kind):
    wl = synth.CONFIGS["c1"]
    plan, exact, size = run_case(fc, oracle, cuda, wl.width, wl.height, wl.num_frames, wl.gop_start, kind,
                                 seed=wl.seed, sample_fps=2.0)
    assert plan.grid_thw == (4, 20, 28)
    assert exact == size  # bit-exact expected


@pytest.mark.parametrize("shape", [
    (64, 48, 28, 56),      # tiny downscale to one merge block row
    (200, 120, 56, 84),    # ragged: 3 merge-block columns (partial strip)
    (96, 40, 56, 140),     # upscale horizontally + vertically
    (224, 224, 224, 224),  # identity (no resample pass in Pillow)
    (854, 480, 476, 840),  # c5 tie case, 15 merge-block columns
    (1280, 720, 560, 1008),
    (1920, 1080, 224, 224),  # paper eval setting: 8.6x downscale, 37-tap filter
    (30, 18, 56, 56),      # odd-size-ish small frame, heavy upscale
])
@pytest.mark.parametrize("kind", ["natural", "uniform"])
def test_shapes(fc, oracle, cuda, kernel, shape, kind):
    W, H, h2, w2 = shape
    N = 8
    plan, exact, size = run_case(fc, oracle, cuda, W, H, N, [0], kind, seed=11,
                                 sampling="explicit", explicit_indices=list(range(0, 8, 2)),
                                 resized_height=h2, resized_width=w2)
    assert plan.resized == (h2, w2)


def test_odd_count_pads_last_frame(fc, oracle, cuda, kernel):
    # 5 explicit frames -> padded to 6 with the last one
    plan, exact, size = run_case(fc, oracle, cuda, 320, 240, 40, [0, 10, 20, 30], "edges", seed=3,
                                 sampling="explicit", explicit_indices=[1, 9, 17, 25, 33])
    assert plan.pad_frames == 1 and plan.grid_thw[0] == 3


@pytest.mark.parametrize("world", [2, 3, 5])
def test_virtual_ranks_concat_equals_single(fc, oracle, cuda, kernel, world):
    """O12 / P:339: the concatenated rank shards equal the single-GPU result
    (all ranks run on one device; no NCCL)."""
    plan, exact, size = run_case(fc, oracle, cuda, 320, 240, 300, list(range(0, 300, 30)), "natural",
                                 seed=5, world=world, sample_fps=2.0)
    assert exact == size


def test_virtual_ranks_odd_explicit(fc, oracle, cuda, kernel):
    # method-b tails and last-rank padding together
    plan, exact, size = run_case(fc, oracle, cuda, 256, 144, 100, list(range(0, 100, 10)), "uniform",
                                 seed=9, world=4, sampling="explicit",
                                 explicit_indices=[0, 3, 12, 13, 14, 25, 41, 42, 57, 70, 81])
    rps = plan.ranks()
    assert rps[-1]["pad_frames"] + sum(r["pad_frames"] for r in rps[:-1]) == 1


# ------------------------------------------------------------ full configs
NCPU = len(os.sched_getaffinity(0))


def _full_config(fc, oracle, cuda, name, kind="natural", clip=0, chunk=30, expect_kernel="tc", backend="pil"):
    """A BASELINE config in the bench's launch configuration (one fc_preprocess
    launch over all frames), compared element by element on the WHOLE token
    tensor with the threaded oracle, chunk pairs at a time."""
    import torch
    wl = synth.CONFIGS[name]
    plan = fc.Plan(fc.VideoMeta(wl.width, wl.height, wl.num_frames, wl.fps, wl.gop_start),
                   fc.ModelCfg(world_size=1, sample_fps=wl.sample_fps, backend=backend))
    idx = plan.sampled_indices
    host = synth.frames_nv12(wl, idx, kind, clip=clip)
    dev = synth.to_device(host)
    surf = fc.SurfaceTable.from_tensors(dev, wl.num_frames)
    tokens = fc.preprocess(plan, 0, surf)
    torch.cuda.synchronize()
    if expect_kernel:
        assert fc.last_kernel() == expect_kernel
    gt, gh, gw = plan.grid_thw
    rpp = gh * gw
    h2, w2 = plan.resized
    exact_total = size_total = 0
    for t0 in range(0, gt, chunk):
        t1 = min(gt, t0 + chunk)
        fr = [idx[min(k, len(idx) - 1)] for k in range(2 * t0, 2 * t1)]
        ref = oracle.preprocess([host[f] for f in fr], wl.width, wl.height, w2, h2, nthreads=NCPU, backend=backend)
        got = tokens[t0 * rpp:t1 * rpp].cpu().numpy()
        exact_total += tol_check(got, ref, f"{name} pairs [{t0}, {t1})")
        size_total += got.size
    assert size_total == plan.token_rows * 1176
    return plan, exact_total, size_total


def _sample_pairs(gt):  # (name kept for the variant tests) every pair of the request
    return range(gt)


def test_full_c1(fc, oracle, cuda, kernel):
    plan, e, s = _full_config(fc, oracle, cuda, "c1", expect_kernel=kernel)
    assert plan.grid_thw == (4, 20, 28) and e == s


def test_full_c2_whole_tensor(fc, oracle, cuda, kernel):
    plan, e, s = _full_config(fc, oracle, cuda, "c2", expect_kernel=kernel)
    assert plan.grid_thw == (60, 40, 72)
    assert e == s


def test_full_c4_whole_tensor(fc, oracle, cuda, kernel):
    plan, e, s = _full_config(fc, oracle, cuda, "c4", kind="edges", expect_kernel=kernel)
    assert plan.grid_thw == (30, 40, 72)
    assert e == s


def test_full_c3_whole_tensor(fc, oracle, cuda, kernel):
    plan, e, s = _full_config(fc, oracle, cuda, "c3", chunk=50, expect_kernel=kernel)
    assert plan.grid_thw == (300, 40, 72)
    assert e == s


def test_full_c5_clip(fc, oracle, cuda, kernel):
    plan, e, s = _full_config(fc, oracle, cuda, "c5", kind="uniform", clip=17, expect_kernel=kernel)
    assert plan.grid_thw == (10, 34, 60)
    assert e == s


# ------------------------------------------------------------ batch launches
def _clip_inputs(fc, wl, clip, kind, plan):
    host = synth.frames_nv12(wl, plan.sampled_indices, kind, clip=clip)
    dev = synth.to_device(host)
    return host, dev, fc.SurfaceTable.from_tensors(dev, wl.num_frames)


def test_batch_homogeneous_matches_oracle(fc, oracle, cuda, kernel):
    """fc_preprocess_batch, config-5 shape: 6 clips with different content in
    ONE launch (per-job token bases, tensor maps in device memory); every
    clip equals the oracle on its own frames."""
    import torch
    wl = synth.CONFIGS["c5"]
    jobs, hosts = [], []
    for clip in range(6):
        plan = fc.Plan(fc.VideoMeta(wl.width, wl.height, wl.num_frames, wl.fps, wl.gop_start),
                       fc.ModelCfg(sampling="explicit", explicit_indices=[3 * clip, 40 + clip, 100, 299 - clip]))
        host, dev, surf = _clip_inputs(fc, wl, clip, "natural" if clip % 2 else "uniform", plan)
        jobs.append((plan, 0, surf, dev))
        hosts.append(host)
    outs = fc.preprocess_batch([(p, r, s) for p, r, s, _ in jobs])
    torch.cuda.synchronize()
    h2, w2 = jobs[0][0].resized
    for (plan, _, _, _), host, out in zip(jobs, hosts, outs):
        ref = oracle.preprocess([host[i] for i in plan.sampled_indices], wl.width, wl.height, w2, h2)
        assert tol_check(out.cpu().numpy(), ref, "batch clip") == ref.size


def test_batch_heterogeneous_equals_single_calls(fc, oracle, cuda, kernel):
    """Mixed shapes, pair counts, a rank with no rows and a job past the
    inline tensor-map limit in one batch call: each job's tokens equal its own
    fc_preprocess call bit for bit (runs of equal geometry share a launch)."""
    import torch
    specs = [  # (W, H, N, gops, cfg, rank)
        (320, 240, 120, [0], dict(sample_fps=2.0), 0),
        (320, 240, 120, [0], dict(sample_fps=2.0), 0),
        (320, 240, 120, [0], dict(sample_fps=2.0, world_size=2), 1),   # no rows
        (320, 240, 120, [0], dict(sampling="explicit", explicit_indices=[1, 7, 9]), 0),
        (200, 120, 16, [0], dict(sampling="explicit", explicit_indices=list(range(16))), 0),
        (64, 48, 300, list(range(0, 300, 30)), dict(sampling="explicit", explicit_indices=list(range(0, 300, 2))), 0),
    ]
    jobs, singles = [], []
    for k, (W, H, N, gops, cfg, rank) in enumerate(specs):
        plan = fc.Plan(fc.VideoMeta(W, H, N, (30, 1), gops), fc.ModelCfg(**cfg))
        host = {i: synth.frame_nv12(W, H, i, "uniform", 50 + k) for i in plan.sampled_indices}
        dev = synth.to_device(host)
        surf = fc.SurfaceTable.from_tensors(dev, N)
        jobs.append((plan, rank, surf, dev))
        singles.append(fc.preprocess(plan, rank, surf) if plan.rank(rank)["row_end"] > plan.rank(rank)["row_begin"]
                       else None)
    outs = fc.preprocess_batch([(p, r, s) for p, r, s, _ in jobs])
    torch.cuda.synchronize()
    for k, (single, out) in enumerate(zip(singles, outs)):
        if single is None:
            assert out.shape[0] == 0
            continue
        assert torch.equal(out.view(torch.int32), single.view(torch.int32)), f"job {k}"
    # the long job (150 frames > inline limit) against the oracle on two pairs
    plan, _, _, _ = jobs[-1]
    W, H = 64, 48
    h2, w2 = plan.resized
    rpp = plan.grid_thw[1] * plan.grid_thw[2]
    idx = plan.sampled_indices
    for t in (0, plan.grid_thw[0] - 1):
        fr = [idx[2 * t], idx[2 * t + 1]]
        ref = oracle.preprocess([synth.frame_nv12(W, H, f, "uniform", 55) for f in fr], W, H, w2, h2)
        tol_check(outs[-1][t * rpp:(t + 1) * rpp].cpu().numpy(), ref, f"long job pair {t}")


def test_full_c5_batch_64_clips(fc, oracle, cuda, kernel):
    """Config 5 as the bench runs it: 64 clips, one fc_preprocess_batch call;
    every clip compared element by element with the oracle."""
    import torch
    wl = synth.CONFIGS["c5"]
    meta = fc.VideoMeta(wl.width, wl.height, wl.num_frames, wl.fps, wl.gop_start)
    plan = fc.Plan(meta, fc.ModelCfg(sample_fps=wl.sample_fps))
    idx = plan.sampled_indices
    jobs = []
    for clip in range(wl.clips):
        host = synth.frames_nv12(wl, idx, "natural", clip=clip)
        dev = synth.to_device(host)
        jobs.append((plan, 0, fc.SurfaceTable.from_tensors(dev, wl.num_frames), dev))
    outs = fc.preprocess_batch([(p, r, s) for p, r, s, _ in jobs])
    torch.cuda.synchronize()
    h2, w2 = plan.resized
    for clip in range(wl.clips):  # every clip, every element
        host = synth.frames_nv12(wl, idx, "natural", clip=clip)
        ref = oracle.preprocess([host[i] for i in idx], wl.width, wl.height, w2, h2, nthreads=NCPU)
        assert tol_check(outs[clip].cpu().numpy(), ref, f"c5 clip {clip}") == ref.size


# ------------------------------------------------------ NEXT-4 variants
@pytest.mark.parametrize("color", ["bt709", "bt601_full", "bt709_full"])
@pytest.mark.parametrize("kind", ["uniform", "edges"])
def test_colour_variants(fc, oracle, cuda, kernel, color, kind):
    """R15: the colour-matrix variants, RGB intermediates and tokens vs the oracle."""
    plan, exact, size = run_case(fc, oracle, cuda, 320, 240, 40, [0, 20], kind, seed=13,
                                 sampling="explicit", explicit_indices=[1, 9, 22, 33], color=color)
    assert exact == size


def _bf16_case(fc, oracle, W, H, N, gops, kind, seed, h2w2=None, **cfg):
    import torch
    extra = dict(resized_height=h2w2[0], resized_width=h2w2[1]) if h2w2 else {}
    plan = fc.Plan(fc.VideoMeta(W, H, N, (30, 1), gops), fc.ModelCfg(token_dtype="bf16", **cfg, **extra))
    idx = plan.sampled_indices
    host = {i: synth.frame_nv12(W, H, i, kind, seed) for i in idx}
    dev = synth.to_device(host)
    surf = fc.SurfaceTable.from_tensors(dev, N)
    out = fc.preprocess(plan, 0, surf)
    torch.cuda.synchronize()
    assert out.dtype == torch.bfloat16 and out.shape == (plan.token_rows, 1176)
    h2, w2 = plan.resized
    ref = oracle.preprocess([host[i] for i in idx], W, H, w2, h2, matrix=cfg.get("color", "bt601"))
    got = out.view(torch.int16).cpu().numpy().view(np.uint16)
    np.testing.assert_array_equal(got, oracle.to_bf16(ref))


@pytest.mark.parametrize("shape", [(320, 240, None), (200, 120, (56, 84)), (1920, 1080, (224, 224))])
def test_bf16_tokens(fc, oracle, cuda, shape):
    """R16: bf16 tokens == RNE(oracle fp32 tokens), bit for bit (ragged strip,
    the paper's 224x224 eval size, and a colour variant on top)."""
    W, H, hw = shape
    _bf16_case(fc, oracle, W, H, 30, [0, 15], "uniform", 17, hw, sampling="explicit",
               explicit_indices=[0, 4, 15, 29, 7][:4] if W != 200 else [0, 4, 15])
    _bf16_case(fc, oracle, W, H, 30, [0, 15], "natural", 18, hw, sampling="explicit",
               explicit_indices=[2, 3], color="bt709")


def test_bf16_full_c2(fc, oracle, cuda):
    """bf16 at BASELINE config 2 in the bench's launch configuration; every pair."""
    import torch
    wl = synth.CONFIGS["c2"]
    plan = fc.Plan(fc.VideoMeta(wl.width, wl.height, wl.num_frames, wl.fps, wl.gop_start),
                   fc.ModelCfg(sample_fps=wl.sample_fps, token_dtype="bf16"))
    idx = plan.sampled_indices
    host = synth.frames_nv12(wl, idx, "natural")
    surf = fc.SurfaceTable.from_tensors(synth.to_device(host), wl.num_frames)
    out = fc.preprocess(plan, 0, surf)
    torch.cuda.synchronize()
    rpp = plan.grid_thw[1] * plan.grid_thw[2]
    h2, w2 = plan.resized
    for t in _sample_pairs(plan.grid_thw[0]):
        ref = oracle.preprocess([host[idx[2 * t]], host[idx[2 * t + 1]]], wl.width, wl.height, w2, h2, nthreads=NCPU)
        got = out[t * rpp:(t + 1) * rpp].view(torch.int16).cpu().numpy().view(np.uint16)
        np.testing.assert_array_equal(got, oracle.to_bf16(ref), err_msg=f"pair {t}")


def test_bf16_debug_dumps_rejected(fc, cuda):
    plan = fc.Plan(fc.VideoMeta(64, 48, 8, (30, 1), [0]),
                   fc.ModelCfg(token_dtype="bf16", sampling="explicit", explicit_indices=[0, 1]))
    host = {i: synth.frame_nv12(64, 48, i, "uniform", 1) for i in (0, 1)}
    surf = fc.SurfaceTable.from_tensors(synth.to_device(host), 8)
    with pytest.raises(fc.FcError) as e:
        fc.preprocess_debug(plan, 0, surf)
    assert e.value.name == "FC_ERR_UNSUPPORTED"


# ------------------------------------------------------ NEXT-1 u8 exchange
def _codes_case(fc, oracle, W, H, N, gops, world, kind, seed, **cfg):
    import torch
    plan = fc.Plan(fc.VideoMeta(W, H, N, (30, 1), gops), fc.ModelCfg(world_size=world, token_dtype="u8", **cfg))
    idx = plan.sampled_indices
    host = {i: synth.frame_nv12(W, H, i, kind, seed) for i in idx}
    surf = fc.SurfaceTable.from_tensors(synth.to_device(host), N)
    parts = [fc.preprocess(plan, r, surf) for r in range(world) if plan.rank(r)["row_end"] > plan.rank(r)["row_begin"]]
    codes = torch.cat(parts, 0)  # what the u8 gather assembles on the encoder
    torch.cuda.synchronize()
    assert codes.dtype == torch.uint8 and codes.shape == (plan.token_rows, 1176)
    h2, w2 = plan.resized
    ref_tok, _, ref_rs = oracle.preprocess([host[i] for i in idx], W, H, w2, h2, want_rgb=True)
    np.testing.assert_array_equal(codes.cpu().numpy(), oracle.codes_from_resized(ref_rs))
    tok = fc.expand_tokens(plan, codes)
    tok16 = fc.expand_tokens(plan, codes, out_dtype="bf16")
    torch.cuda.synchronize()
    np.testing.assert_array_equal(tok.cpu().numpy().view(np.uint32), ref_tok.view(np.uint32))
    np.testing.assert_array_equal(tok16.view(torch.int16).cpu().numpy().view(np.uint16), oracle.to_bf16(ref_tok))


@pytest.mark.parametrize("world", [1, 3])
def test_u8_codes_exchange_and_expand(fc, oracle, cuda, world):
    """NEXT-1: u8 codes per rank (concatenated as the gather would) == the
    oracle's resized values in token layout; fc_expand_tokens of them == the
    oracle's fp32 tokens (and their bf16 rounding) bit for bit."""
    _codes_case(fc, oracle, 320, 240, 300, list(range(0, 300, 30)), world, "natural", 31, sample_fps=2.0)
    _codes_case(fc, oracle, 200, 120, 100, list(range(0, 100, 10)), world, "uniform", 32, sampling="explicit",
                explicit_indices=[0, 3, 12, 13, 14, 25, 41, 42, 57, 70, 81])


def test_u8_codes_full_c2(fc, oracle, cuda):
    """Config 2 through the u8 path (one launch) + expand, every pair vs the oracle."""
    import torch
    wl = synth.CONFIGS["c2"]
    plan = fc.Plan(fc.VideoMeta(wl.width, wl.height, wl.num_frames, wl.fps, wl.gop_start),
                   fc.ModelCfg(sample_fps=wl.sample_fps, token_dtype="u8"))
    idx = plan.sampled_indices
    host = synth.frames_nv12(wl, idx, "natural")
    surf = fc.SurfaceTable.from_tensors(synth.to_device(host), wl.num_frames)
    tok = fc.expand_tokens(plan, fc.preprocess(plan, 0, surf))
    torch.cuda.synchronize()
    rpp = plan.grid_thw[1] * plan.grid_thw[2]
    h2, w2 = plan.resized
    for t in _sample_pairs(plan.grid_thw[0]):
        ref = oracle.preprocess([host[idx[2 * t]], host[idx[2 * t + 1]]], wl.width, wl.height, w2, h2, nthreads=NCPU)
        np.testing.assert_array_equal(tok[t * rpp:(t + 1) * rpp].cpu().numpy().view(np.uint32), ref.view(np.uint32))


# ------------------------------------------------------ NEXT-2 paged output
def _paged_request(fc, W, H, N, gops, seed, token_dtype, **cfg):
    plan = fc.Plan(fc.VideoMeta(W, H, N, (30, 1), gops), fc.ModelCfg(token_dtype=token_dtype, **cfg))
    host = {i: synth.frame_nv12(W, H, i, "natural", seed) for i in plan.sampled_indices}
    dev = synth.to_device(host)
    return plan, fc.SurfaceTable.from_tensors(dev, N), host, dev


def _pool_rows(pool, page_ids, first, n, page_rows):
    """Linear-buffer view of a write chunk: row i -> page_ids[s // R], row s % R."""
    import torch
    idx = [page_ids[(first + i) // page_rows] * page_rows + (first + i) % page_rows for i in range(n)]
    return pool.view(-1, 1176)[torch.tensor(idx, device=pool.device)]


@pytest.mark.parametrize("token_dtype", ["f32", "bf16"])
def test_paged_two_requests_interleaved_pages(fc, oracle, cuda, token_dtype):
    """NEXT-2 (Fig. 10): two requests write into one pool through
    interleaved, non-contiguous page lists, starting mid-page
    (pv_cu_page_len mod page_rows != 0).  Each request reads back exactly its
    single-GPU tokens (differential test vs a linear buffer, SPEC embed_buffer);
    every other pool row keeps its sentinel."""
    import torch
    import random
    R = 64
    tdt = torch.float32 if token_dtype == "f32" else torch.bfloat16
    a = _paged_request(fc, 320, 240, 60, [0, 30], 41, token_dtype, sampling="explicit", explicit_indices=[0, 7, 31, 44])
    b = _paged_request(fc, 200, 120, 40, [0], 42, token_dtype, sampling="explicit", explicit_indices=[1, 2, 3])
    first_a, first_b = 5, 60
    need_a = -(-(first_a + a[0].token_rows) // R)
    need_b = -(-(first_b + b[0].token_rows) // R)
    P = need_a + need_b + 4
    perm = list(range(P))
    random.Random(10).shuffle(perm)  # interleaved, non-contiguous page lists
    ids_a, ids_b = perm[0::2][:need_a], perm[1::2][:need_b]
    assert len(ids_a) == need_a and len(ids_b) == need_b and not set(ids_a) & set(ids_b)
    pool = torch.full((P, R, 1176), -7.0, dtype=tdt, device="cuda")
    fc.preprocess_paged(a[0], 0, a[1], pool, ids_a, first_a)
    fc.preprocess_paged(b[0], 0, b[1], pool, ids_b, first_b)
    torch.cuda.synchronize()
    written = torch.zeros(P * R, dtype=torch.bool)
    for (plan, _, host, _), ids, first in ((a, ids_a, first_a), (b, ids_b, first_b)):
        W, H = plan.meta.width, plan.meta.height
        h2, w2 = plan.resized
        ref = oracle.preprocess([host[i] for i in plan.sampled_indices], W, H, w2, h2)
        got = _pool_rows(pool, ids, first, plan.token_rows, R)
        if token_dtype == "f32":
            np.testing.assert_array_equal(got.cpu().numpy().view(np.uint32), ref.view(np.uint32))
        else:
            np.testing.assert_array_equal(got.view(torch.int16).cpu().numpy().view(np.uint16), oracle.to_bf16(ref))
        for i in range(plan.token_rows):
            written[ids[(first + i) // R] * R + (first + i) % R] = True
    rest = pool.view(-1, 1176)[~written.to(pool.device)]
    assert bool((rest == -7.0).all())


def test_paged_full_c2_matches_linear(fc, cuda):
    """Config 2 through the paged epilogue (page_rows 128, shuffled pages) ==
    the linear fc_preprocess output, bit for bit."""
    import random
    import torch
    wl = synth.CONFIGS["c2"]
    plan = fc.Plan(fc.VideoMeta(wl.width, wl.height, wl.num_frames, wl.fps, wl.gop_start),
                   fc.ModelCfg(sample_fps=wl.sample_fps))
    surf = fc.SurfaceTable.from_tensors(synth.to_device(synth.frames_nv12(wl, plan.sampled_indices, "natural")),
                                        wl.num_frames)
    lin = fc.preprocess(plan, 0, surf)
    R = 128
    npages = -(-(plan.token_rows + 37) // R)
    ids = list(range(npages + 5))
    random.Random(7).shuffle(ids)
    ids = ids[:npages]
    pool = torch.zeros((npages + 5, R, 1176), dtype=torch.float32, device="cuda")
    fc.preprocess_paged(plan, 0, surf, pool, ids, 37)
    torch.cuda.synchronize()
    got = _pool_rows(pool, ids, 37, plan.token_rows, R)
    assert torch.equal(got.view(torch.int32), lin.view(torch.int32))


# ------------------------------------------------------ more edge cases
def test_8k_input_wide_windows(fc, oracle, cuda, kernel):
    """7680x4320 -> smart_resize: ~5.9x downscale, 24+-tap windows, strips whose
    source span needs two TMA boxes per row (NX = 2); one pair vs the oracle."""
    plan, exact, size = run_case(fc, oracle, cuda, 7680, 4320, 8, [0], "natural", seed=77, check_rgb=False,
                                 sampling="explicit", explicit_indices=[2, 5])
    assert plan.max_taps[0] >= 20 and exact == size


def test_cuda_graph_capture_replay(fc, oracle, cuda, kernel):
    """fc_preprocess (tensor maps in the kernel parameters, <= 120 frames) is
    stream-capturable: a captured graph replays to the same tokens, and
    replays after the NV12 surfaces change pick up the new content."""
    import torch
    W, H, N = 320, 240, 120
    plan = make_plan(fc, W, H, N, [0], sample_fps=2.0)
    idx = plan.sampled_indices
    dev = synth.to_device({i: synth.frame_nv12(W, H, i, "natural", 3) for i in idx})
    surf = fc.SurfaceTable.from_tensors(dev, N)
    out = torch.empty((plan.token_rows, 1176), dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    fc.preprocess(plan, 0, surf, out, stream=s)  # warm-up outside capture (tables, maps)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fc.preprocess(plan, 0, surf, out, stream=s)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    h2, w2 = plan.resized
    host2 = {i: synth.frame_nv12(W, H, i, "uniform", 4) for i in idx}
    ref1 = oracle.preprocess([synth.frame_nv12(W, H, i, "natural", 3) for i in idx], W, H, w2, h2)
    np.testing.assert_array_equal(out.cpu().numpy().view(np.uint32), ref1.view(np.uint32))
    for i in idx:  # new content in the same surfaces
        dev[i][0].copy_(torch.from_numpy(host2[i][0]))
        dev[i][1].copy_(torch.from_numpy(host2[i][1]))
    g.replay()
    torch.cuda.synchronize()
    ref2 = oracle.preprocess([host2[i] for i in idx], W, H, w2, h2)
    np.testing.assert_array_equal(out.cpu().numpy().view(np.uint32), ref2.view(np.uint32))


# ------------------------------------------------------ I420 surfaces
@pytest.mark.parametrize("shape", [(320, 240, None), (1920, 1080, None), (3840, 2160, None), (200, 120, (56, 84)),
                                   (1920, 1080, (224, 224))])
@pytest.mark.parametrize("kind", ["uniform", "edges"])
def test_i420_surfaces(fc, oracle, cuda, shape, kind):
    """Planar YUV420 (I420) surfaces: Y + separate U and V planes with their
    own pitch (3 TMA maps per frame).  RGB intermediates bit-exact and tokens
    vs the oracle's I420 path; incl. 4K (two TMA boxes per row)."""
    W, H, h2w2 = shape
    extra = dict(resized_height=h2w2[0], resized_width=h2w2[1]) if h2w2 else {}
    plan = make_plan(fc, W, H, 40, [0, 20], sampling="explicit", explicit_indices=[1, 9, 22, 33, 35],
                     surface_format="i420", **extra)
    idx = plan.sampled_indices
    host = {i: synth.nv12_to_i420(*synth.frame_nv12(W, H, i, kind, 17), W, noise_seed=i) for i in idx}
    surf = fc.SurfaceTable.from_tensors(synth.to_device(host), 40)
    h2, w2 = plan.resized
    ref_tok, ref_src, ref_rs = oracle.preprocess_i420([host[i] for i in idx], W, H, w2, h2, want_rgb=True)
    tok, src, rs = fc.preprocess_debug(plan, 0, surf)
    cuda.cuda.synchronize()
    np.testing.assert_array_equal(src.cpu().numpy(), ref_src[list(range(5)) + [4]])
    np.testing.assert_array_equal(rs.cpu().numpy(), ref_rs[list(range(5)) + [4]])
    got = tok.cpu().numpy()
    assert tol_check(got, ref_tok, f"i420 {W}x{H}") == got.size


def test_i420_full_c2_bench_launch(fc, oracle, cuda):
    """c2 (60 s 1080p, 120 frames) from I420 surfaces in the bench's launch
    configuration (one launch, strip-synchronous mapping), sampled pairs vs
    the oracle."""
    import torch
    wl = synth.CONFIGS["c2"]
    plan = fc.Plan(fc.VideoMeta(wl.width, wl.height, wl.num_frames, wl.fps, wl.gop_start),
                   fc.ModelCfg(surface_format="i420"))
    idx = plan.sampled_indices
    host = {i: synth.nv12_to_i420(*f, wl.width, noise_seed=i)
            for i, f in synth.frames_nv12(wl, idx, "natural").items()}
    surf = fc.SurfaceTable.from_tensors(synth.to_device(host), wl.num_frames)
    out = fc.preprocess(plan, 0, surf)
    torch.cuda.synchronize()
    h2, w2 = plan.resized
    rpp = plan.token_rows // plan.grid_thw[0]
    for t in (0, 29, 59):
        ref = oracle.preprocess_i420([host[idx[2 * t]], host[idx[2 * t + 1]]], wl.width, wl.height, w2, h2)
        assert tol_check(out[t * rpp:(t + 1) * rpp].cpu().numpy(), ref, f"c2 i420 pair {t}") == ref.size


# ------------------------------------------------------ NEXT-1 column split
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_colsplit_virtual_ranks(fc, oracle, cuda, world):
    """fc_preprocess_colsplit ("split along the last dimension"): for
    every rank of a W-way plan (all on this device), block j of its output is
    columns [j*C, (j+1)*C) of its rows of the single-GPU tokens, bit for bit
    (C = 147 for W = 8: blocks start mid-patch); fc_scatter_columns at W = 1
    is the identity."""
    import torch
    W_, H_, N = 320, 240, 300
    plan = make_plan(fc, W_, H_, N, list(range(0, 300, 30)), world, sample_fps=2.0)
    idx = plan.sampled_indices
    host = {i: synth.frame_nv12(W_, H_, i, "natural", 5) for i in idx}
    surf = fc.SurfaceTable.from_tensors(synth.to_device(host), N)
    h2, w2 = plan.resized
    ref = oracle.preprocess([host[i] for i in idx], W_, H_, w2, h2)
    C = 1176 // world
    for r, rp in enumerate(plan.ranks()):
        if rp["row_end"] == rp["row_begin"]:
            continue
        blocks = fc.preprocess_colsplit(plan, r, surf)
        torch.cuda.synchronize()
        assert blocks.shape == (world, rp["row_end"] - rp["row_begin"], C)
        got = blocks.cpu().numpy()
        for j in range(world):
            exp = ref[rp["row_begin"]:rp["row_end"], j * C:(j + 1) * C]
            np.testing.assert_array_equal(got[j].view(np.uint32), np.ascontiguousarray(exp).view(np.uint32),
                                          err_msg=f"rank {r} block {j}")
        if world == 1:
            mine = fc.scatter_columns(plan, 0, None, blocks)
            torch.cuda.synchronize()
            np.testing.assert_array_equal(mine.cpu().numpy().view(np.uint32), ref.view(np.uint32))


# ------------------------------------------------------ a10 exchange, executed
def test_gather_world1_copies_shard(fc, oracle, cuda):
    """fc_gather at W = 1 (no communicator): the encoder's full buffer receives
    the shard through the library's own schedule (one local transfer), bit for
    bit; u8 codes take the same path with 1-byte elements."""
    import torch
    for tok in ("f32", "u8"):
        plan = make_plan(fc, 320, 240, 120, [0], sample_fps=2.0, token_dtype=tok)
        host = {i: synth.frame_nv12(320, 240, i, "natural", 8) for i in plan.sampled_indices}
        surf = fc.SurfaceTable.from_tensors(synth.to_device(host), 120)
        shard = fc.preprocess(plan, 0, surf)
        full = fc.gather(plan, 0, None, shard)
        torch.cuda.synchronize()
        assert full.data_ptr() != shard.data_ptr() and torch.equal(full, shard)
        assert fc.exchange_schedule(plan, 0) == [dict(peer=0, dir="local", src_offset=0, dst_offset=0,
                                                      bytes=shard.numel() * shard.element_size())]


def test_tc_kernel_serves_the_baseline_configs(fc, cuda, monkeypatch):
    """With FC_TC=1 the tcgen05 kernel's plan fits every BASELINE config
    (c1-c5); the paper's 224x224 setting (37-tap windows) falls to the mma.sync
    kernel; without it the mma.sync kernel serves everything."""
    import torch
    monkeypatch.setenv("FC_TC", "1")
    for name in ("c1", "c2", "c3", "c4", "c5"):
        wl = synth.CONFIGS[name]
        plan = fc.Plan(fc.VideoMeta(wl.width, wl.height, wl.num_frames, wl.fps, wl.gop_start),
                       fc.ModelCfg(sampling="explicit", explicit_indices=[0, 1]))
        host = {i: synth.frame_nv12(wl.width, wl.height, i, "natural", 1) for i in (0, 1)}
        fc.preprocess(plan, 0, fc.SurfaceTable.from_tensors(synth.to_device(host), wl.num_frames))
        torch.cuda.synchronize()
        assert fc.last_kernel() == "tc", name
    plan = make_plan(fc, 1920, 1080, 8, [0], sampling="explicit", explicit_indices=[0, 1], resized_height=224,
                     resized_width=224)
    host = {i: synth.frame_nv12(1920, 1080, i, "natural", 1) for i in (0, 1)}
    fc.preprocess(plan, 0, fc.SurfaceTable.from_tensors(synth.to_device(host), 8))
    torch.cuda.synchronize()
    assert fc.last_kernel() == "mma"
    monkeypatch.delenv("FC_TC")
    wl = synth.CONFIGS["c1"]
    plan = fc.Plan(fc.VideoMeta(wl.width, wl.height, wl.num_frames, wl.fps, wl.gop_start),
                   fc.ModelCfg(sampling="explicit", explicit_indices=[0, 1]))
    host = {i: synth.frame_nv12(wl.width, wl.height, i, "natural", 1) for i in (0, 1)}
    fc.preprocess(plan, 0, fc.SurfaceTable.from_tensors(synth.to_device(host), wl.num_frames))
    torch.cuda.synchronize()
    assert fc.last_kernel() == "mma"


def test_submit_equals_plan_then_preprocess(fc, oracle, cuda):
    """fc_submit (plan + launch in one call) gives the oracle's tokens, and its
    plan equals fc_plan's; a bad surface table leaves nothing enqueued."""
    import torch
    wl = synth.CONFIGS["c1"]
    meta = fc.VideoMeta(wl.width, wl.height, wl.num_frames, wl.fps, wl.gop_start)
    cfg = fc.ModelCfg(sample_fps=wl.sample_fps)
    ref_plan = fc.Plan(meta, cfg)
    idx = ref_plan.sampled_indices
    host = synth.frames_nv12(wl, idx, "uniform")
    surf = fc.SurfaceTable.from_tensors(synth.to_device(host), wl.num_frames)
    out = torch.full((ref_plan.token_rows, 1176), -1.0, device="cuda")
    plan = fc.submit(meta, cfg, 0, surf, out)
    torch.cuda.synchronize()
    assert plan.sampled_indices == idx and plan.grid_thw == ref_plan.grid_thw
    h2, w2 = plan.resized
    ref = oracle.preprocess([host[i] for i in idx], wl.width, wl.height, w2, h2)
    assert tol_check(out.cpu().numpy(), ref, "fc_submit") == ref.size
    bad = fc.SurfaceTable(wl.num_frames)  # every surface NULL
    out.fill_(-1.0)
    with pytest.raises(fc.FcError) as e:
        fc.submit(meta, cfg, 0, bad, out)
    assert e.value.name == "FC_ERR_MISSING_SURFACE"
    torch.cuda.synchronize()
    assert bool((out == -1.0).all())


# ------------------------------------------- NEXT-4 torchvision backend (R21)
@pytest.mark.parametrize("shape", [(320, 240, None), (1920, 1080, None), (3840, 2160, None), (854, 480, None),
                                   (200, 120, (56, 84)), (1920, 1080, (224, 224))])
@pytest.mark.parametrize("kind", ["uniform", "edges"])
def test_torchvision_backend_shapes(fc, oracle, cuda, kernel, shape, kind):
    """HF torchvision-backend arithmetic (torch uint8 AA bicubic at its int16
    precision, fused normalisation): RGB intermediates bit-exact and tokens vs
    the oracle, through the debug and the production instance."""
    W, H, hw = shape
    cfg = dict(sampling="explicit", explicit_indices=[0, 7, 19], backend="torchvision")
    if hw:
        cfg.update(resized_height=hw[0], resized_width=hw[1])
    plan, exact, size = run_case(fc, oracle, cuda, W, H, 30, [0, 15], kind, seed=29, **cfg)
    assert exact == size


def test_torchvision_backend_virtual_ranks(fc, oracle, cuda, kernel):
    plan, exact, size = run_case(fc, oracle, cuda, 640, 360, 300, list(range(0, 300, 30)), "natural", seed=5,
                                 world=3, backend="torchvision")
    assert exact == size


def test_torchvision_backend_full_c2(fc, oracle, cuda, kernel):
    plan, e, s = _full_config(fc, oracle, cuda, "c2", expect_kernel=kernel, backend="torchvision")
    assert plan.grid_thw == (60, 40, 72) and e == s


def test_torchvision_backend_full_c4(fc, oracle, cuda, kernel):
    plan, e, s = _full_config(fc, oracle, cuda, "c4", kind="uniform", expect_kernel=kernel, backend="torchvision")
    assert e == s


def test_torchvision_backend_bf16_and_codes(fc, oracle, cuda):
    """bf16 tokens and u8 codes + fc_expand_tokens take the backend's table."""
    import torch
    W, H = 320, 240
    for td in ("bf16", "u8"):
        plan = make_plan(fc, W, H, 30, [0, 15], sampling="explicit", explicit_indices=[2, 11, 20, 29],
                         backend="torchvision", token_dtype=td)
        idx = plan.sampled_indices
        host = {i: synth.frame_nv12(W, H, i, "uniform", 31, synth.pitch_for(W)) for i in idx}
        surf = fc.SurfaceTable.from_tensors(synth.to_device(host), 30)
        h2, w2 = plan.resized
        ref = oracle.preprocess([host[i] for i in idx], W, H, w2, h2, backend="torchvision")
        out = fc.preprocess(plan, 0, surf)
        torch.cuda.synchronize()
        if td == "bf16":
            np.testing.assert_array_equal(out.view(torch.int16).cpu().numpy().view(np.uint16), oracle.to_bf16(ref))
        else:
            tok = fc.expand_tokens(plan, out, out_dtype="f32")
            torch.cuda.synchronize()
            assert tol_check(tok.cpu().numpy(), ref, "codes expanded") == ref.size
