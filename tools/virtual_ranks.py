"""Per-rank preprocess latency of a request split over W GPUs, measured on ONE
GPU by running each rank's launch of the W-way plan in turn (virtual ranks):
the compute half of the multi-GPU latency (max over ranks), with no exchange.
This pod's boxes have one GPU, so this is the only N>1 number measurable here;
it is not a scaling run.

    python tools/virtual_ranks.py [config] [reps]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_17574_b200 as fc  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
wl = synth.CONFIGS[name]
meta = fc.VideoMeta(wl.width, wl.height, wl.num_frames, wl.fps, wl.gop_start)
plan1 = fc.Plan(meta, fc.ModelCfg(sample_fps=wl.sample_fps))
dev = synth.to_device(synth.frames_nv12(wl, plan1.sampled_indices, "natural"))
surf = fc.SurfaceTable.from_tensors(dev, wl.num_frames)
res = {"workload": name, "method": "each rank's launch of the W-way plan run alone on one B200, CUDA events, "
                                    f"mean of {reps}; latency = max over ranks (exchange not included)"}
for W in (1, 2, 4, 8):
    for tok in ("f32", "u8"):
        plan = fc.Plan(meta, fc.ModelCfg(world_size=W, sample_fps=wl.sample_fps, token_dtype=tok))
        per = []
        for r in range(W):
            rows = plan.rank_rows(r)
            if not rows:
                per.append(0.0)
                continue
            out = torch.empty((rows, 1176), dtype=torch.float32 if tok == "f32" else torch.uint8, device="cuda")
            for _ in range(3):
                fc.preprocess(plan, r, surf, out)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                fc.preprocess(plan, r, surf, out)
            e1.record()
            torch.cuda.synchronize()
            per.append(e0.elapsed_time(e1) / reps)
        res[f"W{W}_{tok}"] = {"max_ms": round(max(per), 4), "per_rank_ms": [round(x, 4) for x in per],
                              "pairs": [(plan.rank(r)["sampled_count"] + plan.rank(r)["pad_frames"]) // 2
                                        for r in range(W)]}
print(json.dumps(res))
