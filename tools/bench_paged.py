"""NEXT-2 read_chunk bandwidth: fc_paged_copy gathering an iteration's tokens
from a paged pool into a contiguous chunk ("materialise them into
contiguous memory only at use time").

The pool holds c2's token rows (172,800 fp32 rows of 4704 B = 812.9 MB, larger
than L2) in 128-row pages in shuffled order, split over 8 requests.  Two
chunk sizes: the paper's encode token budget (10,240 tokens per iteration,
P:690) and a whole request.  Each timed launch reads a different part of the
pool (so reads come from HBM); CUDA events around K launches on the current
stream, queued behind a GPU sleep so the host's enqueue cost (reported
separately as host_us_per_call) is off the device timeline; algorithmic
bytes = 2 x rows x 4704 (read + write).

    python tools/bench_paged.py [reps]
"""
import ctypes
import json
import os
import random
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_17574_b200 as fc  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]
P, ROWS, NREQ, COLS = 128, 172_800, 8, 1176
pages = -(-ROWS // P) + NREQ
rng = random.Random(1)
per = ROWS // NREQ
# the table hands out pages lowest id first; the kernel only sees ids, so a
# fixed permutation of them stands for a pool fragmented by earlier requests
perm = list(range(pages))
rng.shuffle(perm)
pool = torch.empty((pages, P, COLS), dtype=torch.float32, device="cuda")
pool.view(torch.int32).random_()

res = {"pool_rows": ROWS, "page_rows": P, "pool_bytes": pool.numel() * 4, "peak_gbs": peak}
for name, chunk_rows in (("encode_chunk_10240", 10240), ("whole_request_21600", per)):
    # NREQ-way split of each iteration's budget, starting at a rotating offset
    idxs = []
    tab = fc.PageTable(pages, P)
    for r in range(NREQ):
        tab.alloc(r, per)
    tab.index("write", list(range(NREQ)), [per] * NREQ)
    read = [0] * NREQ
    for it in range(reps + 3):
        counts = [0] * NREQ
        if chunk_rows >= per:
            r = it % NREQ
            if read[r] + per > per:
                break
            counts[r] = per
        else:
            left = chunk_rows
            for r in range(NREQ):
                c = min(left, per - read[r], chunk_rows // NREQ + 1)
                counts[r] = c
                left -= c
            if sum(counts) < chunk_rows:
                break
        idx = tab.index("read", list(range(NREQ)), counts)
        idx.pv_page_indices = [perm[p] for p in idx.pv_page_indices]
        for r in range(NREQ):
            read[r] += counts[r]
        idxs.append(idx)
    chunk = torch.empty((max(sum(i.pv_indptr[-1] for i in idxs[:1]), 1), COLS), dtype=torch.float32, device="cuda")
    L = fc.lib()
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    cs = [idx.to_c() for idx in idxs]  # marshalled once: the C call is what is timed on the host

    def launch(c):
        fc._native.check(L.fc_paged_copy(1, ctypes.byref(c[0]), ctypes.c_void_p(pool.data_ptr()), pages, P,
                                         COLS * 4, ctypes.c_void_p(chunk.data_ptr()), stream), "fc_paged_copy")
    for c in cs[:3]:
        launch(c)
    timed = cs[3:]
    if not timed:
        continue
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(4_000_000)  # ~2 ms: the host enqueues every launch before the first runs
    e0.record()
    h0 = time.perf_counter()
    for c in timed:
        launch(c)
    host_us = (time.perf_counter() - h0) / len(timed) * 1e6
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / len(timed)
    timed = idxs[3:]
    rows = timed[0].pv_indptr[-1]
    gbs = 2 * rows * COLS * 4 / ms / 1e6
    res[name] = {"rows": rows, "launches": len(timed), "ms": round(ms, 5), "gbs": round(gbs, 1),
                 "frac": round(gbs / peak, 3), "blocks_per_launch": len(timed[0].pv_page_indices),
                 "host_us_per_call": round(host_us, 1)}
print(json.dumps(res))
