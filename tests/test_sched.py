"""Stall-free GOP_s dispatch (Alg. 2) through the C ABI,
CPU only: the decode callback sleeps, so the scheduling invariants are checked
on their own (a decode unit = one admitted segment)."""
import random
import threading
import time

import pytest


class Recorder:
    def __init__(self, durations):
        self.d = durations
        self.lock = threading.Lock()
        self.active = 0
        self.max_active = 0
        self.events = []  # (t, kind, segment, worker)

    def __call__(self, seg, w):
        with self.lock:
            self.active += 1
            self.max_active = max(self.max_active, self.active)
            self.events.append((time.perf_counter(), "start", seg, w))
        time.sleep(self.d[seg])
        with self.lock:
            self.active -= 1
            self.events.append((time.perf_counter(), "end", seg, w))
        return 0


@pytest.mark.parametrize("T,N", [(3, 1), (4, 2), (8, 3), (2, 4)])
def test_gate_order_and_coverage(fc, T, N):
    rng = random.Random(T * 10 + N)
    nseg = 4 * T
    worker_of = [rng.randrange(T) for _ in range(nseg)]
    rec = Recorder([rng.uniform(0.002, 0.01) for _ in range(nseg)])
    trace = fc.dispatch_segments(worker_of, T, N, rec)
    assert sorted(s for s, _, _ in trace) == list(range(nseg))            # every segment exactly once
    assert all(worker_of[s] == w and st == 0 for s, w, st in trace)       # on its own worker
    assert rec.max_active <= N                                            # at most N decode units busy (l.10)
    for w in range(T):                                                    # a worker's segments in order
        mine = [s for s, ww, _ in trace if ww == w]
        assert mine == sorted(mine)


def test_same_worker_keeps_its_unit(fc):
    """N = 1: a worker that finishes a segment and has more dispatches its next
    one before any waiting worker (l.12-13), so execution is worker-contiguous."""
    T = 4
    worker_of = [i % T for i in range(4 * T)]
    trace = fc.dispatch_segments(worker_of, T, 1, lambda s, w: (time.sleep(0.002), 0)[1])
    ws = [w for _, w, _ in trace]
    runs = [ws[0]] + [b for a, b in zip(ws, ws[1:]) if a != b]
    assert len(runs) == T and sorted(runs) == list(range(T))


def test_segment_granularity_removes_the_stall(fc):
    """Fig. 9 (right): 4 units, two videos of very unequal length.  Whole-video
    scheduling (one task per video) leaves two units idle and waits for the long
    video; GOP_s segments dealt over 4 workers keep all units busy."""
    unit = 0.004
    long_v, short_v = 24, 4   # GOP_s segments per video, each `unit` long
    t0 = time.perf_counter()
    fc.dispatch_segments([0, 1], 2, 4, lambda s, w: (time.sleep(unit * (long_v if s == 0 else short_v)), 0)[1])
    whole = time.perf_counter() - t0
    segs = long_v + short_v
    t0 = time.perf_counter()
    fc.dispatch_segments([i % 4 for i in range(segs)], 4, 4, lambda s, w: (time.sleep(unit), 0)[1])
    stall_free = time.perf_counter() - t0
    assert stall_free < 0.6 * whole, (stall_free, whole)


def test_failure_stops_dispatch(fc):
    started = []
    lock = threading.Lock()

    def fn(s, w):
        with lock:
            started.append(s)
        time.sleep(0.002)
        return 7 if s == 2 else 0
    with pytest.raises(fc.FcError, match="FC_ERR_CUDA"):
        fc.dispatch_segments([0] * 6, 1, 1, fn)
    assert started == [0, 1, 2]   # nothing after the failed segment on that worker


def test_argument_errors(fc):
    import ctypes
    L = fc.lib()
    cb = fc._native.SEGMENT_FN(lambda c, s, w: 0)
    wo = (ctypes.c_int32 * 2)(0, 5)
    assert fc._native.STATUS[L.fc_dispatch_segments(wo, 2, 2, 1, cb, None, None)] == "FC_ERR_INVALID_ARG"
    assert fc._native.STATUS[L.fc_dispatch_segments(wo, 1, 0, 1, cb, None, None)] == "FC_ERR_INVALID_ARG"
    assert fc._native.STATUS[L.fc_dispatch_segments(wo, 1, 1, 0, cb, None, None)] == "FC_ERR_INVALID_ARG"
    assert fc._native.STATUS[L.fc_dispatch_segments(None, 0, 1, 1, cb, None, None)] == "FC_OK"
    assert fc._native.STATUS[L.fc_decode_mjpeg(None, None, 3, None, 1, 1, 1, 0, None)] == "FC_ERR_INVALID_ARG"
