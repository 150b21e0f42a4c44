"""NEXT-4 JPEG images ("JPEG is decoded via dedicated hardware"):
nvJPEG decodes into I420 planes, the fused kernel turns them into tokens.

The decoder is library code, so it is only sanity-pinned (its luma against
libjpeg's through Pillow, within the IDCT rounding difference; its RGB against
Pillow's decode); the parity bar starts at the decoded planes: tokens from
fc.preprocess_jpeg == the oracle's I420 path (full-range BT.601, R15) on the
same planes copied to the host, bit for bit."""
import io

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


def _jpeg(rgb: np.ndarray, subsampling: int = 2, quality: int = 90) -> bytes:
    from PIL import Image
    buf = io.BytesIO()
    Image.fromarray(rgb).save(buf, "JPEG", quality=quality, subsampling=subsampling)
    return buf.getvalue()


def _image(W, H, seed):
    y, uv = synth.frame_nv12(W, H, seed, "natural", seed)
    from oracle import oracle as o
    return o.nv12_to_rgb(y, uv, W, H)


@pytest.fixture(scope="module")
def decoder(fc, cuda):
    d = fc.JpegDecoder("auto")
    print(f"nvJPEG backend: {d.backend} {d.hardware_error}")
    yield d
    d.close()


@pytest.mark.parametrize("wh", [(640, 480), (1920, 1080), (300, 200)])
def test_decode_sanity_vs_libjpeg(fc, cuda, decoder, wh):
    from PIL import Image
    W, H = wh
    data = _jpeg(_image(W, H, 3))
    assert decoder.info(data) == (W, H, True)
    y, u, v = decoder.decode(data)
    cuda.cuda.synchronize()
    im = Image.open(io.BytesIO(data))
    im.draft("YCbCr", im.size)
    ycc = np.asarray(im.convert("YCbCr") if im.mode != "YCbCr" else im)
    d = np.abs(y[:, :W].cpu().numpy().astype(int) - ycc[..., 0].astype(int))
    assert d.max() <= 2 and (d > 0).mean() < 0.05, (d.max(), (d > 0).mean())
    # chroma: the 2x2 block means of libjpeg's (fancy-upsampled) Cb/Cr stay close to nvJPEG's planes
    cb = ycc[..., 1].astype(float).reshape(H // 2, 2, W // 2, 2).mean(axis=(1, 3))
    assert np.abs(u[:, :W // 2].cpu().numpy() - cb).mean() < 2.0


@pytest.mark.parametrize("case", [(640, 480, {}), (1920, 1080, {}), (300, 200, {"resized_height": 224, "resized_width": 224}),
                                  (1280, 720, {"min_pixels": 56 * 56, "max_pixels": 28 * 28 * 1280})])
def test_jpeg_tokens_match_oracle(fc, oracle, cuda, decoder, case):
    import torch
    W, H, kw = case
    data = _jpeg(_image(W, H, 11))
    tokens, grid, plan, (y, u, v) = fc.preprocess_jpeg(decoder, data, fc.image_cfg(**kw))
    torch.cuda.synchronize()
    h2, w2 = plan.resized
    assert grid == (1, h2 // 14, w2 // 14) and tokens.shape == (grid[1] * grid[2], 1176)
    host = (y.cpu().numpy(), u.cpu().numpy(), v.cpu().numpy())
    ref = oracle.preprocess_i420([host], W, H, w2, h2, matrix="bt601_full")
    got = tokens.cpu().numpy()
    np.testing.assert_array_equal(got.view(np.uint32), ref.view(np.uint32))
    # the decoded image's RGB (oracle, nearest chroma) is close to Pillow's decode (fancy upsampling)
    from PIL import Image
    rgb_pil = np.asarray(Image.open(io.BytesIO(data)).convert("RGB")).astype(int)
    ref_tok, ref_src, _ = oracle.preprocess_i420([host], W, H, w2, h2, matrix="bt601_full", want_rgb=True)
    assert np.abs(ref_src[0].astype(int) - rgb_pil).mean() < 3.0


def test_jpeg_unsupported_inputs(fc, cuda, decoder):
    rgb = _image(320, 240, 5)
    with pytest.raises(fc.FcError, match="UNSUPPORTED"):
        decoder.decode(_jpeg(rgb, subsampling=0))            # 4:4:4
    with pytest.raises(fc.FcError, match="UNSUPPORTED"):
        decoder.decode(_jpeg(np.ascontiguousarray(rgb[:, :317])))  # odd width
    with pytest.raises(fc.FcError):
        decoder.decode(b"\xff\xd8not a jpeg at all" * 4)
    assert decoder.info(_jpeg(rgb, subsampling=0))[2] is False


def test_mjpeg_stall_free_decode_matches_single_decodes(fc, oracle, cuda, decoder):
    """NEXT-3 (partial): a Motion-JPEG request (every frame an independent
    JPEG, a one-frame GOP) decoded over GOP_s segments by 3 workers with at
    most 2 in flight (Alg. 2): each target's planes equal a single decode, and
    the request's tokens equal the oracle on those planes."""
    import torch
    W, H = 640, 360
    frames = [_jpeg(_image(W, H, 40 + i)) for i in range(10)]
    planes, trace = fc.decode_mjpeg(frames, segments=5, workers=3, max_in_flight=2)
    assert sorted(s for s, _, _ in trace) == list(range(5)) and all(st == 0 for _, _, st in trace)
    for i, f in enumerate(frames):
        ref = decoder.decode(f)
        torch.cuda.synchronize()
        for a, b, wv in zip(planes[i], ref, (W, W // 2, W // 2)):  # visible bytes (pitch padding is unset)
            assert torch.equal(a[:, :wv], b[:, :wv])
    plan = fc.Plan(fc.VideoMeta(W, H, len(frames), (30, 1), [0]),
                   fc.image_cfg(sampling="fps_stride", explicit_indices=None, sample_fps=30.0, min_frames=2))
    surf = fc.SurfaceTable(len(frames))
    for i in plan.sampled_indices:
        surf.set(i, *planes[i])
    tokens = fc.preprocess(plan, 0, surf)
    torch.cuda.synchronize()
    h2, w2 = plan.resized
    host = [tuple(p.cpu().numpy() for p in planes[i]) for i in plan.sampled_indices]
    ref = oracle.preprocess_i420(host, W, H, w2, h2, matrix="bt601_full")
    np.testing.assert_array_equal(tokens.cpu().numpy().view(np.uint32), ref.view(np.uint32))
