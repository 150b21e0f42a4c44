import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2512_17574_b200 as fc
import synth
W, H = int(sys.argv[1]), int(sys.argv[2])
plan = fc.Plan(fc.VideoMeta(W, H, 40, (30, 1), [0, 20]), fc.ModelCfg(sampling="explicit", explicit_indices=[1, 9], surface_format="i420"))
host = {i: synth.nv12_to_i420(*synth.frame_nv12(W, H, i, "uniform", 17), W, noise_seed=i) for i in plan.sampled_indices}
for k, v in host.items(): print(k, [p.shape for p in v])
surf = fc.SurfaceTable.from_tensors(synth.to_device(host), 40)
out = fc.preprocess(plan, 0, surf)
torch.cuda.synchronize()
print("ok", out.shape)
