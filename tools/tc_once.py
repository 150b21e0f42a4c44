"""One fc_preprocess launch of a BASELINE config (compute-sanitizer / debugging)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("FC_TC", "1")  # the tcgen05 kernel
import torch  # noqa: E402

import paper_2512_17574_b200 as fc  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
wl = synth.CONFIGS[name]
npairs = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg = fc.ModelCfg(sample_fps=wl.sample_fps)
plan = fc.Plan(fc.VideoMeta(wl.width, wl.height, wl.num_frames, wl.fps, wl.gop_start), cfg)
idx = plan.sampled_indices
if npairs:
    plan = fc.Plan(fc.VideoMeta(wl.width, wl.height, wl.num_frames, wl.fps, wl.gop_start),
                   fc.ModelCfg(sampling="explicit", explicit_indices=idx[:2 * npairs]))
    idx = plan.sampled_indices
dev = synth.to_device(synth.frames_nv12(wl, idx, "natural"))
surf = fc.SurfaceTable.from_tensors(dev, wl.num_frames)
out = fc.preprocess(plan, 0, surf)
torch.cuda.synchronize()
print(name, "ok", fc.last_kernel(), out.shape)
