"""Multi-process host logic of the N>1 path on CPU (gloo, world size 2/3).

One process per rank, as bench.py runs under torchrun.  Each rank builds the
plan independently (it must be identical on every rank: no coordination is
needed, the plan is a pure function of the request), computes ITS shard -- here
with the CPU oracle, since this box has no GPU -- and runs the library's own
exchange schedule (fc_exchange_schedule: exactly the transfers fc_gather /
fc_scatter_columns hand to NCCL) with gloo isend/irecv on byte buffers.  The
receiver checks the P:339 invariant: the assembled result equals the
single-GPU result bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q, exchange="f32"):
    import sys
    sys.path.insert(0, ROOT)
    import hashlib

    import torch
    import torch.distributed as dist

    import paper_2512_17574_b200 as fc
    import synth
    from oracle import oracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        W, H, N, gops, cfg = case
        tok = "u8" if exchange == "u8" else "f32"  # the plan's token dtype sizes the exchanged rows
        plan = fc.Plan(fc.VideoMeta(W, H, N, (30, 1), gops), fc.ModelCfg(world_size=world, token_dtype=tok, **cfg))
        # 1) every rank derived the same plan
        digest = hashlib.sha256(repr((plan.sampled_indices, plan.ranks(), plan.grid_thw)).encode()).digest()
        mine = torch.tensor(list(digest), dtype=torch.uint8)
        allg = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(allg, mine)
        assert all(torch.equal(a, mine) for a in allg), "plans differ between ranks"
        # 2) this rank's shard (oracle stands in for the device kernel on CPU)
        rp = plan.rank(rank)
        idx = plan.sampled_indices
        frames = idx[rp["sampled_begin"]:rp["sampled_begin"] + rp["sampled_count"]]
        frames += [frames[-1]] * rp["pad_frames"] if frames else []
        h2, w2 = plan.resized
        host = {i: synth.frame_nv12(W, H, i, "natural", 21) for i in set(frames)}
        rows = rp["row_end"] - rp["row_begin"]
        if exchange == "u8":  # NEXT-1: ship the u8 codes, expand on the encoder
            shard = (oracle.codes_from_resized(oracle.preprocess([host[f] for f in frames], W, H, w2, h2,
                                                                 want_rgb=True)[2]) if frames
                     else np.zeros((0, 1176), np.uint8))
        else:
            shard = (oracle.preprocess([host[f] for f in frames], W, H, w2, h2) if frames
                     else np.zeros((0, 1176), np.float32))
        assert shard.shape[0] == rows
        host_all = {i: synth.frame_nv12(W, H, i, "natural", 21) for i in idx}
        ref = oracle.preprocess([host_all[i] for i in idx], W, H, w2, h2)
        enc = plan.cfg.encoder_rank
        if exchange == "colsplit":  # NEXT-1 column split: all-to-all of column blocks
            C = 1176 // world
            blocks = np.stack([shard[:, j * C:(j + 1) * C] for j in range(world)]) if rows else np.zeros((world, 0, C))
            send = torch.from_numpy(np.ascontiguousarray(blocks, dtype=np.float32).reshape(-1).view(np.uint8))
            recv = torch.zeros(plan.token_rows * C * 4, dtype=torch.uint8)
            kind = "colsplit"
        else:
            send = torch.from_numpy(np.ascontiguousarray(shard).reshape(-1).view(np.uint8))
            recv = torch.zeros(plan.token_rows * 1176 * shard.itemsize if rank == enc else 0, dtype=torch.uint8)
            kind = "gather"
        # 3) the library's schedule over the process group (fc_gather / fc_scatter_columns' transfers)
        reqs = []
        for x in fc.exchange_schedule(plan, rank, kind):
            a, b, n = x["src_offset"], x["dst_offset"], x["bytes"]
            if x["dir"] == "local":
                recv[b:b + n] = send[a:a + n]
            elif x["dir"] == "send":
                reqs.append(dist.isend(send[a:a + n].clone(), x["peer"]))
            else:
                buf = torch.empty(n, dtype=torch.uint8)
                reqs.append((dist.irecv(buf, x["peer"]), buf, b))
        for rq in reqs:
            if isinstance(rq, tuple):
                rq[0].wait()
                recv[rq[2]:rq[2] + len(rq[1])] = rq[1]
            else:
                rq.wait()
        if exchange == "colsplit":
            assert recv.numpy().tobytes() == \
                np.ascontiguousarray(ref[:, rank * C:(rank + 1) * C]).view(np.uint32).tobytes(), "column slice"
        elif rank == enc:
            full = recv.numpy().view(shard.dtype).reshape(plan.token_rows, 1176)
            if exchange == "u8":  # expand: R5 table per channel of each column
                lut = np.array([[oracle.normalize_value(v, c) for v in range(256)] for c in range(3)], np.float32)
                full = lut[(np.arange(1176) // 392)[None, :], full]
            assert full.view(np.uint32).tobytes() == ref.view(np.uint32).tobytes(), "gathered != single-GPU result"
        q.put((rank, "ok"))
    except Exception as e:  # report to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


CASES = [
    (320, 240, 300, list(range(0, 300, 30)), dict(sample_fps=2.0)),
    (256, 144, 100, list(range(0, 100, 10)),
     dict(sampling="explicit", explicit_indices=[0, 3, 12, 13, 14, 25, 41, 42, 57, 70, 81])),
    (320, 240, 120, [0], dict(sample_fps=2.0)),  # single GOP: all on the encoder, other ranks idle
]


def _run(world, case, exchange):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, CASES[case], q, exchange)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {r: "ok" for r in range(world)}, res


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_gloo_gather_equals_single_gpu(world, case):
    _run(world, case, "f32")


@pytest.mark.parametrize("case", [0, 1])
def test_gloo_u8_exchange_equals_single_gpu(case):
    """NEXT-1 exchange: u8 codes gathered (4x fewer bytes) and expanded on the
    encoder give the single-GPU fp32 tokens bit for bit."""
    _run(3, case, "u8")


@pytest.mark.parametrize("world,case", [(2, 0), (3, 1), (3, 2)])
def test_gloo_column_split_equals_single_gpu_columns(world, case):
    """NEXT-1 column split (fc_scatter_columns' row arithmetic):
    after the all-to-all, rank j holds columns [j*C, (j+1)*C) of the
    single-GPU tokens, every row, bit for bit (incl. idle ranks, case 2)."""
    _run(world, case, "colsplit")
