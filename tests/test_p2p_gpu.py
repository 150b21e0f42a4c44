"""NEXT-1 fused peer-store exchange: a rank's
kernel writes its token rows straight into the encoder's buffer through a CUDA
IPC mapping, so there is no separate gather pass.

This pod's boxes have one GPU, so both "ranks" are separate processes on
cuda:0: the encoder process exports its full token buffer (fc_ipc_export_range),
the other process maps it (fc_ipc_import) and runs fc_preprocess for its rank
with tokens = peer base + row_begin * row bytes.  On an 8-GPU box the same
stores cross NVLink.  The encoder then checks the P:339 invariant: the buffer
equals the single-GPU result bit for bit (and, for u8 codes, after its own
expand)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _case():
    return 320, 240, 300, list(range(0, 300, 30))


def _peer(handle, offset, tok, q_done):
    import sys
    sys.path.insert(0, ROOT)
    import torch

    import paper_2512_17574_b200 as fc
    import synth
    try:
        torch.cuda.set_device(0)
        W, H, N, gops = _case()
        plan = fc.Plan(fc.VideoMeta(W, H, N, (30, 1), gops), fc.ModelCfg(world_size=2, sample_fps=2.0, token_dtype=tok))
        rp = plan.rank(1)
        rows = rp["row_end"] - rp["row_begin"]
        fr = plan.sampled_indices[rp["sampled_begin"]:rp["sampled_begin"] + rp["sampled_count"]]
        surf = fc.SurfaceTable.from_tensors(synth.to_device({i: synth.frame_nv12(W, H, i, "natural", 23) for i in fr}), N)
        peer = fc.PeerBuffer(handle)
        dt = {"f32": torch.float32, "u8": torch.uint8}[tok]
        esz = 4 if tok == "f32" else 1
        view = peer.tensor((rows, 1176), dt, offset + rp["row_begin"] * 1176 * esz)
        fc.preprocess(plan, 1, surf, view)  # the epilogue stores land in the encoder's buffer
        torch.cuda.synchronize()
        peer.close()
        q_done.put("ok")
    except Exception as e:  # report to the encoder process
        q_done.put(repr(e))


@pytest.mark.parametrize("tok", ["f32", "u8"])
def test_peer_store_exchange_equals_single_gpu(fc, oracle, cuda, tok):
    import torch
    import torch.multiprocessing as mp

    import synth
    W, H, N, gops = _case()
    plan = fc.Plan(fc.VideoMeta(W, H, N, (30, 1), gops), fc.ModelCfg(world_size=2, sample_fps=2.0, token_dtype=tok))
    assert plan.rank(1)["row_end"] > plan.rank(1)["row_begin"]  # both ranks have rows
    dt = {"f32": torch.float32, "u8": torch.uint8}[tok]
    full = torch.full((plan.token_rows, 1176), 7, dtype=dt, device="cuda")
    handle, offset = fc.ipc_export(full)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_peer, args=(handle, offset, tok, q))
    p.start()
    # rank 0 (the encoder) writes its own rows in place
    rp0 = plan.rank(0)
    fr0 = plan.sampled_indices[rp0["sampled_begin"]:rp0["sampled_begin"] + rp0["sampled_count"]]
    surf0 = fc.SurfaceTable.from_tensors(synth.to_device({i: synth.frame_nv12(W, H, i, "natural", 23) for i in fr0}), N)
    fc.preprocess(plan, 0, surf0, full[rp0["row_begin"]:rp0["row_end"]])
    torch.cuda.synchronize()
    res = q.get(timeout=180)
    p.join(timeout=60)
    assert res == "ok", res
    idx = plan.sampled_indices
    h2, w2 = plan.resized
    frames = [synth.frame_nv12(W, H, i, "natural", 23) for i in idx]
    ref_tok, _, ref_rs = oracle.preprocess(frames, W, H, w2, h2, want_rgb=True)
    if tok == "f32":
        np.testing.assert_array_equal(full.cpu().numpy().view(np.uint32), ref_tok.view(np.uint32))
    else:
        np.testing.assert_array_equal(full.cpu().numpy(), oracle.codes_from_resized(ref_rs))
        tokens = fc.expand_tokens(plan, full)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(tokens.cpu().numpy().view(np.uint32), ref_tok.view(np.uint32))
