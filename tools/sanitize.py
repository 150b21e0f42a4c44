"""Small runs of every kernel path for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): the tcgen05 kernel (fp32 + debug, batch, >120-frame
launch) and the mma.sync kernel (the same with FC_TC=0, plus bf16, u8 codes,
paged output incl. first_offset 0 with rows a multiple of the page size,
column split, I420 surfaces) and fc_expand_tokens."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_17574_b200 as fc  # noqa: E402
import synth  # noqa: E402


def run(W, H, N, gops, **cfg):
    plan = fc.Plan(fc.VideoMeta(W, H, N, (30, 1), gops), fc.ModelCfg(**cfg))
    host = {i: synth.frame_nv12(W, H, i, "natural", 3) for i in plan.sampled_indices}
    if cfg.get("surface_format") == "i420":
        host = {i: synth.nv12_to_i420(y, uv, W, noise_seed=i) for i, (y, uv) in host.items()}
    dev = synth.to_device(host)
    surf = fc.SurfaceTable.from_tensors(dev, N)
    return plan, surf, dev


def common():
    plan, surf, _ = run(320, 240, 120, [0], sample_fps=2.0)
    fc.preprocess(plan, 0, surf)
    fc.preprocess_debug(plan, 0, surf)
    jobs = [run(256, 144, 60, [0, 30], sample_fps=2.0) for _ in range(3)]
    fc.preprocess_batch([(p, 0, s) for p, s, _ in jobs])
    planL, surfL, _ = run(64, 48, 300, list(range(0, 300, 30)), sampling="explicit",
                          explicit_indices=list(range(0, 260, 2)))
    fc.preprocess(planL, 0, surfL)  # 130 frames: tensor maps in the device descriptor
    plan3, surf3, _ = run(1280, 720, 60, [0, 30], sampling="explicit", explicit_indices=[0, 5, 9, 40])
    fc.preprocess(plan3, 0, surf3)
    torch.cuda.synchronize()


common()  # tcgen05 kernel (default for NV12 / fp32)
os.environ["FC_TC"] = "0"
common()  # the same workload through the mma.sync kernel
plan, surf, _ = run(320, 240, 120, [0], sample_fps=2.0)
# paged output: first_offset 0, 2240 rows = 35 pages of 64 (the last thread rows past the write)
pool = torch.zeros((40, 64, 1176), dtype=torch.float32, device="cuda")
fc.preprocess_paged(plan, 0, surf, pool, list(range(35)), 0)
fc.preprocess_paged(plan, 0, surf, pool, list(range(3, 39)), 37)
planC, surfC, _ = run(320, 240, 300, list(range(0, 300, 30)), sample_fps=2.0, world_size=8)
for r in range(8):
    if planC.rank(r)["row_end"] > planC.rank(r)["row_begin"]:
        fc.preprocess_colsplit(planC, r, surfC)
plan16, surf16, _ = run(200, 120, 40, [0, 20], sampling="explicit", explicit_indices=[1, 5, 9], token_dtype="bf16")
fc.preprocess(plan16, 0, surf16)
plan8, surf8, _ = run(320, 240, 120, [0], sample_fps=2.0, token_dtype="u8")
codes = fc.preprocess(plan8, 0, surf8)
fc.expand_tokens(plan8, codes)
fc.expand_tokens(plan8, codes, out_dtype="bf16")
plan224, surf224, _ = run(1920, 1080, 8, [0], sampling="explicit", explicit_indices=[0, 3],
                          resized_height=224, resized_width=224)
fc.preprocess(plan224, 0, surf224)  # KSH=KSV=3, 28-column strips
planI, surfI, _ = run(640, 360, 60, [0, 30], sample_fps=2.0, surface_format="i420")
fc.preprocess(planI, 0, surfI)  # I420: Y, U, V tensor maps
fc.preprocess_debug(planI, 0, surfI)
torch.cuda.synchronize()
print("sanitize workload done")
