"""NEXT-2, the paged embedding buffer (Fig. 10; SPEC
embed_buffer S:218-290; reading R21).

CPU (``-m "not gpu"``): the oracle (oracle/paged.py) against SPEC's worked
examples, the Fig. 10 reconstruction (tests/golden/fig10_pages.txt) and flat
per-request linear buffers; then libfc's page table (fc_pages_*) against the
oracle on the same randomized operation sequences -- every index array, freed
list, counter and error must agree.  GPU: fc_paged_copy (read_chunk /
write_chunk) against the oracle's row-by-row copy, byte for byte, and the
whole path -- fc_preprocess_paged writes, chunked reads with eager free --
against the linear single-request tokens.
"""
import ctypes
import os
import random

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def paged():
    from oracle import paged as p
    return p


# ---------------------------------------------------------------- oracle pins

def test_oracle_spec_alloc_examples(paged):
    b = paged.PagedBuffer(16, 128)
    assert b.alloc(0, 0) == []                     # S:241 tokens=0 -> no pages
    assert b.alloc(1, 300) == [0, 1, 2]            # S:242 ceil(300/128) = 3 pages
    small = paged.PagedBuffer(2, 128)
    with pytest.raises(paged.OutOfPages):          # S:243 pool of 2, needs 3: nothing allocated
        small.alloc(7, 300)
    assert small.free == [0, 1] and small.pages == {}


def test_oracle_spec_write_examples(paged):
    P = 128
    b = paged.PagedBuffer(4, P)
    b.alloc(0, 256)
    idx = b.index("write", [0], [128])             # cu=0, 128 tokens fill page 0 exactly
    assert idx == ([0, 128], [0, 1], [0], [0])
    idx = b.index("write", [0], [1])               # the next write starts at page 1, offset 0
    assert idx == ([0, 1], [0, 1], [1], [128])
    # cu=100, write 56 -> 28 tokens to page A offsets 100..127, 28 to page B offsets 0..27
    c = paged.PagedBuffer(4, P)
    c.alloc(5, 156)
    c.index("write", [5], [100])
    idx = c.index("write", [5], [56])
    rows = list(paged._token_rows(idx, P))
    assert [(p, s) for _, p, s in rows[:28]] == [(0, o) for o in range(100, 128)]
    assert [(p, s) for _, p, s in rows[28:]] == [(1, o) for o in range(28)]
    with pytest.raises(paged.PageError):           # capacity: nothing past the allocated pages
        c.index("write", [5], [101])


def _fig10():
    steps = []
    for line in open(os.path.join(GOLDEN, "fig10_pages.txt")):
        line = line.split("#")[0].strip()
        if line:
            op, *args = line.split()
            steps.append((op, args))
    return steps


class _ProductTable:
    """libfc's page table behind the oracle's method names."""

    def __init__(self, fc, total, P):
        self.t = fc.PageTable(total, P)

    def alloc(self, req, tokens):
        return self.t.alloc(req, tokens)

    def index(self, op, reqs, counts):
        r = self.t.index(op, reqs, counts)
        return r.pv_indptr, r.pv_page_indptr, r.pv_page_indices, r.pv_cu_page_len

    def free_consumed(self):
        return self.t.free_consumed()

    def release(self, req):
        return self.t.release(req)


def _run_fig10(make):
    steps = dict((op, a) for op, a in _fig10() if op in ("page_size", "total_pages"))
    b = make(int(steps["total_pages"][0]), int(steps["page_size"][0]))
    ids = {}
    last_index = None
    for op, args in _fig10():
        pairs = [a.split(":") for a in args]
        if op == "alloc":
            got = {}
            for name, n in pairs:
                ids.setdefault(name, len(ids))
                got[name] = b.alloc(ids[name], int(n))
        elif op == "expect_pages":
            assert {n: [int(x) for x in v.split(",")] for n, v in pairs} == got
        elif op in ("write", "read"):
            last_index = b.index(op, [ids[n] for n, _ in pairs], [int(c) for _, c in pairs])
        elif op == "expect_index":
            want = {k: [int(x) for x in v.split(",")] for k, v in (a.split("=") for a in args)}
            assert list(last_index[0]) == want["pv_indptr"]
            assert list(last_index[1]) == want["pv_page_indptr"]
            assert list(last_index[2]) == want["pv_page_indices"]
            assert list(last_index[3]) == want["pv_cu_page_len"]
        elif op == "expect_freed":
            want = [] if args == ["-"] else [int(x) for x in args[0].split(",")]
            assert sorted(b.free_consumed()) == want


def test_oracle_fig10(paged):
    _run_fig10(lambda total, P: paged.PagedBuffer(total, P))


def _random_ops(rng, total, P, nops):
    """A random alloc / write / read / release / free sequence."""
    ops, live = [], []
    for _ in range(nops):
        k = rng.random()
        if k < 0.25 or not live:
            req = rng.randrange(6)
            ops.append(("alloc", req, rng.randrange(0, 3 * P)))
            if req not in live:
                live.append(req)
        elif k < 0.55:
            reqs = rng.sample(live, rng.randint(1, len(live)))
            ops.append(("write", reqs, [rng.randrange(0, 2 * P) for _ in reqs]))
        elif k < 0.85:
            reqs = rng.sample(live, rng.randint(1, len(live)))
            ops.append(("read", reqs, [rng.randrange(0, 2 * P) for _ in reqs]))
        elif k < 0.93:
            ops.append(("free",))
        else:
            req = live.pop(rng.randrange(len(live)))
            ops.append(("release", req))
    return ops


def _apply(b, op, errors):
    """Run one op on the oracle; returns its result or the error class name."""
    try:
        if op[0] == "alloc":
            return b.alloc(op[1], op[2])
        if op[0] in ("write", "read"):
            return b.index(op[0], op[1], op[2])
        if op[0] == "free":
            return b.free_consumed()
        return b.release(op[1])
    except errors as e:
        return type(e).__name__


def test_oracle_matches_linear_buffers(paged):
    """reads through the pages byte-match flat per-request buffers;
    free + owned + consumed == total after every op; no page freed twice; no
    leak once every request is released."""
    rng = random.Random(20251217)
    for seq in range(150):
        P = rng.choice([1, 2, 4, 8])
        total = rng.randrange(1, 24)
        b = paged.PagedBuffer(total, P)
        pool = np.full((total, P), -1, dtype=np.int64)
        linear: dict[int, list[int]] = {}
        next_tok = 0
        freed_since_alloc = set()
        for op in _random_ops(rng, total, P, rng.randrange(1, 120)):
            if op[0] in ("write", "read"):
                try:
                    idx = b.index(op[0], op[1], op[2])
                except paged.PageError:
                    continue
                if op[0] == "write":
                    chunk = np.arange(next_tok, next_tok + idx[0][-1], dtype=np.int64)
                    next_tok += idx[0][-1]
                    pool = paged.write_chunk(pool, idx, P, chunk)
                    for i, r in enumerate(op[1]):
                        linear.setdefault(r, []).extend(chunk[idx[0][i]:idx[0][i + 1]].tolist())
                else:
                    got = paged.read_chunk(pool, idx, P)
                    for i, r in enumerate(op[1]):
                        start = idx[3][i]
                        want = linear.get(r, [])[start:start + op[2][i]]
                        assert got[idx[0][i]:idx[0][i + 1]].tolist() == want
            elif op[0] == "free":
                out = b.free_consumed()
                assert not (set(out) & freed_since_alloc), "a page freed twice"
                freed_since_alloc |= set(out)
            elif op[0] == "alloc":
                try:
                    new = b.alloc(op[1], op[2])
                except paged.OutOfPages:
                    continue
                freed_since_alloc -= set(new)
            else:
                try:
                    b.release(op[1])
                except paged.PageError:  # its alloc had failed: never known
                    continue
                linear.pop(op[1], None)
            assert len(b.free) + b.owned() + len(b.consumed) == total
            # eager-free optimality: no owned page is fully read
            for r, pages in b.pages.items():
                for g in range(len(pages)):
                    if (g + 1) * P <= b.read[r]:
                        assert g in b.consumed_pages[r]
        for r in list(b.pages):
            b.release(r)
        b.free_consumed()
        assert b.free == list(range(total))  # no leak


# ---------------------------------------------------------------- product vs oracle (host, no GPU)

def test_product_fig10(fc):
    _run_fig10(lambda total, P: _ProductTable(fc, total, P))


def test_product_page_table_matches_oracle(fc, paged):
    rng = random.Random(7)
    for seq in range(200):
        P = rng.choice([1, 2, 4, 8, 16])
        total = rng.randrange(0, 24)
        o = paged.PagedBuffer(total, P)
        g = _ProductTable(fc, total, P)
        for op in _random_ops(rng, total, P, rng.randrange(1, 80)):
            want = _apply(o, op, (paged.OutOfPages, paged.PageError))
            try:
                got = _apply(g, op, ())
                if op[0] in ("write", "read"):
                    got = tuple(list(x) for x in got)
                    want = tuple(list(x) for x in want) if isinstance(want, tuple) else want
            except fc.FcError as e:
                got = {"FC_ERR_OUT_OF_PAGES": "OutOfPages", "FC_ERR_INVALID_ARG": "PageError"}[e.name]
            if op[0] == "release":
                got = want if got is None else got
            assert got == want, (seq, op)
            fr, ow, co, live = g.t.stats()
            assert (fr, ow, co) == (len(o.free), o.owned(), len(o.consumed))
            assert live == len(o.pages)


def test_product_page_table_errors(fc):
    t = fc.PageTable(2, 128)
    with pytest.raises(fc.FcError) as e:
        t.alloc(0, 300)
    assert e.value.name == "FC_ERR_OUT_OF_PAGES"
    assert t.stats() == (2, 0, 0, 0)               # nothing allocated
    assert t.alloc(0, 200) == [0, 1]
    for bad in (lambda: t.index("write", [0], [257]),      # CapacityError
                lambda: t.index("read", [0], [1]),         # UnwrittenRange
                lambda: t.index("write", [0, 0], [1, 1]),  # a request twice
                lambda: t.index("write", [3], [1]),        # no pages
                lambda: t.index("write", [0], [-1]),
                lambda: t.release(9)):
        with pytest.raises(fc.FcError) as e:
            bad()
        assert e.value.name == "FC_ERR_INVALID_ARG"
    assert t.index("write", [0], [0]).pv_page_indices == []
    for args in ((0, 128), (-1, 128), (4, 3), (4, 0)):
        if args == (0, 128):
            fc.PageTable(*args)  # an empty pool is valid
            continue
        with pytest.raises(fc.FcError):
            fc.PageTable(*args)


def test_paged_copy_rejects_bad_index_without_gpu(fc):
    """Validation happens before any CUDA call (runs on a CPU-only host)."""
    from paper_2512_17574_b200 import RaggedIndex, _native
    L = fc.lib()
    bad = [RaggedIndex([0, 5], [0, 1], [0], [0]),     # 5 tokens from offset 0 need 2 pages of 4
           RaggedIndex([0, 2], [0, 1], [9], [0]),     # page outside the pool
           RaggedIndex([1, 2], [0, 1], [0], [0]),     # pv_indptr[0] != 0
           RaggedIndex([0, 2], [0, 1], [0], [-1])]    # negative cu
    for idx in bad:
        c, _keep = idx.to_c()
        st = L.fc_paged_copy(1, ctypes.byref(c), ctypes.c_void_p(16), 4, 4, 64, ctypes.c_void_p(16), None)
        assert _native.STATUS[st] == "FC_ERR_INVALID_ARG"
    c, _keep = RaggedIndex([0, 0], [0, 0], [], [3]).to_c()   # nothing to move: no launch, OK
    assert L.fc_paged_copy(1, ctypes.byref(c), None, 4, 4, 64, None, None) == 0
    c, _keep = RaggedIndex([0, 2], [0, 1], [0], [0]).to_c()
    assert _native.STATUS[L.fc_paged_copy(1, ctypes.byref(c), ctypes.c_void_p(16), 4, 4, 12,
                                          ctypes.c_void_p(16), None)] == "FC_ERR_INVALID_ARG"  # row_bytes % 8


# ---------------------------------------------------------------- GPU: fc_paged_copy and the whole path

def _random_index(rng, paged, total, P, nreq, max_tokens):
    """A valid iteration index over a shuffled pool (the oracle's table)."""
    b = paged.PagedBuffer(total, P)
    b.free = rng.sample(range(total), total)  # non-contiguous page ids
    reqs = list(range(nreq))
    for r in reqs:
        b.alloc(r, rng.randrange(0, max_tokens))
        b.free = sorted(b.free, key=lambda _: rng.random())
    pre = [rng.randrange(0, b.reserved[r] + 1) for r in reqs]   # tokens written in earlier iterations
    b.index("write", reqs, pre)
    counts = [rng.randrange(0, b.reserved[r] - pre[i] + 1) for i, r in enumerate(reqs)]
    return b.index("write", reqs, counts)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,cols", [("float32", 1176), ("bfloat16", 1176), ("uint8", 1176), ("float32", 4)])
@pytest.mark.parametrize("P,nreq,max_tokens,total", [(4, 3, 40, 64), (128, 5, 700, 40), (1, 40, 30, 800)])
def test_paged_copy_vs_oracle(fc, paged, cuda, dtype, cols, P, nreq, max_tokens, total):
    import torch
    from paper_2512_17574_b200 import RaggedIndex
    rng = random.Random(hash((dtype, cols, P, nreq)) & 0xFFFF)
    idx = _random_index(rng, paged, total, P, nreq, max_tokens)
    ri = RaggedIndex(*[list(x) for x in idx])
    tdt = getattr(torch, dtype)
    g = torch.Generator().manual_seed(3)
    pool_h = torch.randint(0, 255, (total, P, cols), generator=g, dtype=torch.uint8).to(tdt)
    rows = idx[0][-1]
    # read_chunk
    pool = pool_h.cuda()
    chunk = torch.full((max(rows, 1), cols), 7, dtype=tdt, device="cuda")
    fc.paged_copy("read", ri, pool, chunk)
    torch.cuda.synchronize()
    want = paged.read_chunk(pool_h.view(torch.uint8 if dtype == "uint8" else torch.int16 if dtype == "bfloat16"
                                        else torch.int32).numpy(), idx, P)
    got = chunk[:rows].cpu().view(torch.uint8 if dtype == "uint8" else torch.int16 if dtype == "bfloat16"
                                  else torch.int32).numpy()
    np.testing.assert_array_equal(got, want)
    # write_chunk: every other pool row keeps its value
    src = torch.randint(0, 255, (max(rows, 1), cols), generator=g, dtype=torch.uint8).to(tdt)
    fc.paged_copy("write", ri, pool, src.cuda())
    torch.cuda.synchronize()
    iv = torch.uint8 if dtype == "uint8" else torch.int16 if dtype == "bfloat16" else torch.int32
    want = paged.write_chunk(pool_h.view(iv).numpy(), idx, P, src.view(iv).numpy())
    np.testing.assert_array_equal(pool.cpu().view(iv).numpy(), want)


@pytest.mark.gpu
def test_paged_copy_many_blocks(fc, paged, cuda):
    """> 320 blocks: the block list travels as a device descriptor."""
    import torch
    from paper_2512_17574_b200 import RaggedIndex
    rng = random.Random(11)
    idx = _random_index(rng, paged, 3000, 2, 60, 90)
    assert len(idx[2]) > 320
    pool_h = torch.randint(-2**31, 2**31 - 1, (3000, 2, 1176), dtype=torch.int32)
    chunk = torch.empty((idx[0][-1], 1176), dtype=torch.int32, device="cuda")
    fc.paged_copy("read", RaggedIndex(*[list(x) for x in idx]), pool_h.cuda(), chunk)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(chunk.cpu().numpy(), paged.read_chunk(pool_h.numpy(), idx, 2))


@pytest.mark.gpu
@pytest.mark.parametrize("tok", ["f32", "bf16"])
def test_paged_buffer_end_to_end(fc, paged, cuda, tok):
    """Two video requests written by fc_preprocess_paged through libfc's page
    table, then consumed by read_chunk in chunks of tau = 700 tokens per
    iteration (the encoder's token budget, P:690 uses 2048): every chunk equals
    the linear single-GPU tokens, and the pages freed after each iteration
    equal the oracle table's."""
    import torch

    import synth
    P = 128
    dt = torch.float32 if tok == "f32" else torch.bfloat16
    reqs = []
    for r, (W, H) in enumerate([(320, 240), (480, 270)]):
        meta = fc.VideoMeta(W, H, 60, (30, 1), list(range(0, 60, 15)))
        plan = fc.Plan(meta, fc.ModelCfg(sample_fps=4.0, token_dtype=tok))
        surf = fc.SurfaceTable.from_tensors(synth.to_device({i: synth.frame_nv12(W, H, i, "natural", 5 + r)
                                                             for i in plan.sampled_indices}), 60)
        linear = fc.preprocess(plan, 0, surf)
        reqs.append((plan, surf, linear))
    total = sum(-(-p.token_rows // P) for p, _, _ in reqs) + 3
    t = fc.PageTable(total, P)
    o = paged.PagedBuffer(total, P)
    pool = torch.zeros((total, P, 1176), dtype=dt, device="cuda")
    for r, (plan, surf, _) in enumerate(reqs):
        assert t.alloc(r, plan.token_rows) == o.alloc(r, plan.token_rows)
    for r, (plan, surf, _) in enumerate(reqs):  # one write chunk per request (the vision worker)
        idx = t.index("write", [r], [plan.token_rows])
        o.index("write", [r], [plan.token_rows])
        fc.preprocess_paged(plan, 0, surf, pool, idx.pv_page_indices, idx.pv_cu_page_len[0] % P)
    read = [0, 0]
    tau = 700
    while read[0] < reqs[0][0].token_rows or read[1] < reqs[1][0].token_rows:
        counts, budget = [], tau
        for r in range(2):
            c = min(budget, reqs[r][0].token_rows - read[r])
            counts.append(c)
            budget -= c
        idx = t.index("read", [0, 1], counts)
        want_idx = o.index("read", [0, 1], counts)
        assert (idx.pv_indptr, idx.pv_page_indptr, idx.pv_page_indices, idx.pv_cu_page_len) == \
            tuple(list(x) for x in want_idx)
        chunk = torch.empty((idx.pv_indptr[-1], 1176), dtype=dt, device="cuda")
        fc.paged_copy("read", idx, pool, chunk)
        torch.cuda.synchronize()
        for r in range(2):
            lin = reqs[r][2][read[r]:read[r] + counts[r]]
            assert torch.equal(chunk[idx.pv_indptr[r]:idx.pv_indptr[r + 1]], lin)
            read[r] += counts[r]
        assert sorted(t.free_consumed()) == sorted(o.free_consumed())
    for r in range(2):
        t.release(r)
        o.release(r)
    t.free_consumed()
    assert t.stats() == (total, 0, 0, 0)
