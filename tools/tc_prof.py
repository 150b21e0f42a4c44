"""One launch of a BASELINE config through the tcgen05 kernel's FC_TC_PROF
instance: per role, the fraction of each warp's lifetime spent in each
barrier wait (printed by libfc to stderr)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("FC_TC", "1")  # the tcgen05 kernel
import torch  # noqa: E402

import paper_2512_17574_b200 as fc  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
wl = synth.CONFIGS[name]
plan = fc.Plan(fc.VideoMeta(wl.width, wl.height, wl.num_frames, wl.fps, wl.gop_start),
               fc.ModelCfg(sample_fps=wl.sample_fps))
dev = synth.to_device(synth.frames_nv12(wl, plan.sampled_indices, "natural"))
surf = fc.SurfaceTable.from_tensors(dev, wl.num_frames)
out = fc.preprocess(plan, 0, surf)
torch.cuda.synchronize()
os.environ["FC_TC_PROF"] = "1"
for abl in [0] + [int(a) for a in sys.argv[2:]]:
    os.environ["FC_TC_ABLATE"] = str(abl)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fc.preprocess(plan, 0, surf, out)
    e1.record()
    torch.cuda.synchronize()
    print(f"{name} ablate {abl}: {e0.elapsed_time(e1):.4f} ms", file=sys.stderr, flush=True)
del os.environ["FC_TC_PROF"]
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    fc.preprocess(plan, 0, surf, out)
e1.record()
torch.cuda.synchronize()
print(f"{name}: {fc.last_kernel()} kernel {e0.elapsed_time(e1) / 10:.4f} ms")
