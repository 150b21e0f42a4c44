export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "u8 or bf16" 2>&1 | tail -2
python - <<'PY'
import torch, synth, paper_2512_17574_b200 as fc
wl = synth.CONFIGS["c2"]
plan = fc.Plan(fc.VideoMeta(wl.width, wl.height, wl.num_frames, wl.fps, wl.gop_start), fc.ModelCfg(token_dtype="u8"))
codes = torch.randint(0, 256, (plan.token_rows, 1176), dtype=torch.uint8, device="cuda")
for dt in ("f32", "bf16"):
    o = torch.empty((plan.token_rows, 1176), dtype=torch.float32 if dt == "f32" else torch.bfloat16, device="cuda")
    for _ in range(5): fc.expand_tokens(plan, codes, o, dt)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): fc.expand_tokens(plan, codes, o, dt)
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    nb = codes.numel() * (1 + (4 if dt == "f32" else 2))
    print(f"expand {dt}: {ms:.4f} ms  {nb / ms / 1e6:.0f} GB/s")
PY
