import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_2512_17574_b200 as fc
wl = synth.CONFIGS["c2"]
plan = fc.Plan(fc.VideoMeta(wl.width, wl.height, wl.num_frames, wl.fps, wl.gop_start), fc.ModelCfg(token_dtype="u8"))
codes = torch.randint(0, 256, (plan.token_rows, 1176), dtype=torch.uint8, device="cuda")
o32 = torch.empty((plan.token_rows, 1176), dtype=torch.float32, device="cuda")
o16 = torch.empty((plan.token_rows, 1176), dtype=torch.bfloat16, device="cuda")
def t(fn, nb, name):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): fn()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    print(f"{name:28s} {ms:.4f} ms  {nb / ms / 1e6:.0f} GB/s")
n = codes.numel()
t(lambda: fc.expand_tokens(plan, codes, o32, "f32"), 5 * n, "expand f32")
t(lambda: fc.expand_tokens(plan, codes, o16, "bf16"), 3 * n, "expand bf16")
t(lambda: o32.copy_(codes), 5 * n, "torch u8->f32 copy_")
t(lambda: o16.copy_(codes), 3 * n, "torch u8->bf16 copy_")
t(lambda: o32.fill_(1.0), 4 * n, "torch fill f32 (write only)")
t(lambda: o32.view(-1)[: n // 2].copy_(o32.view(-1)[n // 2:]), 4 * n, "torch f32 copy (r+w)")
