"""Host-side cost of one small request (config 1) through the Python binding:
fc_plan (Plan), fc_preprocess (enqueue only), and the raw C calls."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_17574_b200 as fc  # noqa: E402
import synth  # noqa: E402

wl = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c1"]
meta = fc.VideoMeta(wl.width, wl.height, wl.num_frames, wl.fps, wl.gop_start)
cfg = fc.ModelCfg(sample_fps=wl.sample_fps)
plan = fc.Plan(meta, cfg)
dev = synth.to_device(synth.frames_nv12(wl, plan.sampled_indices, "natural"))
surf = fc.SurfaceTable.from_tensors(dev, wl.num_frames)
out = fc.preprocess(plan, 0, surf)
torch.cuda.synchronize()


def t(fn, n=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    dt = (time.perf_counter() - t0) / n * 1e6
    torch.cuda.synchronize()
    return dt


m, km = meta.to_c()
c, kc = cfg.to_c()
h = ctypes.c_void_p()
grid = (ctypes.c_int64 * 3)()
sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
optr = ctypes.c_void_p(out.data_ptr())


def raw_plan():
    fc.lib().fc_plan(ctypes.byref(m), ctypes.byref(c), ctypes.byref(h))
    fc.lib().fc_plan_destroy(h)


print(f"Plan() {t(lambda: fc.Plan(meta, cfg)):.1f} us | raw fc_plan+destroy {t(raw_plan):.1f} us | "
      f"preprocess() {t(lambda: fc.preprocess(plan, 0, surf, out)):.1f} us | raw fc_preprocess "
      f"{t(lambda: fc.lib().fc_preprocess(plan.handle, 0, surf.arr, surf.n, optr, grid, sp)):.1f} us")
