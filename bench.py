#!/usr/bin/env python3
"""bench.py -- per-video preprocess latency / frames/s of the FlashCodec hot
path on B200 (BASELINE.json metric), with its HBM roofline and the CPU oracle
beside it.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

N>1 is launched by torchrun (one process per GPU, NCCL).  A "step" is one
pass of the whole hot path over one request:
  a1-a4  fc_plan on the host (sampling, smart_resize, GOP partition, tables)
  a5-a9  fc_preprocess: one fused kernel launch per rank
  a10    fc_gather of the row shards to the encoder rank (N>1)
The host plans request k+1 while the GPU runs request k (all inside the
timed region).  Inputs are resident in HBM when the timed region starts
(`value`); `e2e` repeats the step through the same public API from pinned
host buffers, with the NV12 upload and a device->host read of the result
inside the timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_PATH = os.path.join(ROOT, "profiles", "ncu_traffic.json")
METRIC = "per-video preprocess frames/s (latency = ms_per_step)"


def load_peaks():
    try:
        with open(PEAKS_PATH) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"  # B200_PROFILING.md fallback


def load_traffic(workload: str, key: str = "dram_bytes_per_launch"):
    try:
        with open(TRAFFIC_PATH) as f:
            d = json.load(f)
        return d.get(workload, {}).get(key)
    except Exception:
        return None


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, dev_index: int):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                fn = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                    nv.nvmlDeviceGetCurrentClocksThrottleReasons
                r = fn(self._h)
                for k, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def workload_meta(fc, wl):
    return fc.VideoMeta(wl.width, wl.height, wl.num_frames, wl.fps, wl.gop_start)


def algorithmic_bytes(plan, wl, rank_plan=None, tok_bytes=4):
    """1.5*W*H read per sampled frame + 1176 tokens
    written per token row (4704 B fp32, 2352 B bf16)."""
    if rank_plan is None:
        n = plan.num_sampled
        rows = plan.token_rows
    else:
        n = rank_plan["sampled_count"]
        rows = rank_plan["row_end"] - rank_plan["row_begin"]
    return int(n * 1.5 * wl.width * wl.height + rows * 1176 * tok_bytes)


# ------------------------------------------------------------ CPU oracle arm
def oracle_sample(wl, pairs, nthreads, matrix="bt601", backend="pil"):
    """Run the oracle (as it stands) on `pairs` temporal pairs of workload wl.
    Returns (seconds, frames)."""
    from oracle import oracle
    idx = oracle.sample_indices(wl.num_frames, wl.fps[0] / wl.fps[1], wl.sample_fps)
    take = idx[: 2 * pairs]
    host = synth.frames_nv12(wl, take, "natural")
    h2, w2 = oracle.smart_resize(wl.height, wl.width)
    t0 = time.perf_counter()
    oracle.preprocess([host[i] for i in take], wl.width, wl.height, w2, h2, nthreads=nthreads, matrix=matrix,
                      backend=backend)
    return time.perf_counter() - t0, len(take)


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    wl = synth.CONFIGS[args.config]
    cores = len(os.sched_getaffinity(0))
    # each step is the whole request when (warm-up + timed) steps fit ~2 minutes of
    # host time, else the largest prefix of its temporal pairs that does
    from oracle import oracle
    n_all = len(oracle.sample_indices(wl.num_frames, wl.fps[0] / wl.fps[1], wl.sample_fps))
    gt = (n_all + 1) // 2
    probe = min(gt, max(1, cores // 2))
    dt, _ = oracle_sample(wl, probe, cores)
    per_pair = dt / probe
    pairs = int(max(1, min(gt, 120.0 / max(1, args.steps + args.warmup) / max(per_pair, 1e-6))))
    for _ in range(args.warmup):
        oracle_sample(wl, pairs, cores)
    tot, frames = 0.0, 0
    for _ in range(args.steps):
        dt, f = oracle_sample(wl, pairs, cores)
        tot += dt
        frames += f
    value = frames / tot
    sample = (f"{2 * pairs} sampled frames ({pairs} of {gt} temporal pairs"
              f"{': the whole request' if pairs == gt else ''}) of {args.config} per step, natural content")
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "frames/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(tot / args.steps * 1e3, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u8->f32", "data": "synthetic",
            "config": {"workload": f"{args.config}: {wl.note}", "frames_per_step": 2 * pairs},
            "cpu_baseline": {"value": round(value, 4), "unit": "frames/s", "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": round(value, 4), "unit": "frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2512_17574_b200 as fc

    rank, world, local = dist_env()
    if world != args.gpus:
        print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl = synth.CONFIGS[args.config]
    clips = wl.clips                              # c5: 64 independent requests per step
    meta = workload_meta(fc, wl)
    # throughput mode (c5) at N>1 is "replicas only": whole clips
    # are placed on GPUs by LPT on their pairs (fc_assign_requests), each GPU
    # runs ONE batched launch over its clips, and nothing is exchanged
    replicas = clips > 1 and world > 1
    clip_ids = list(range(clips))
    if replicas:
        pairs = [fc.Plan(meta, fc.ModelCfg(sample_fps=wl.sample_fps)).grid_thw[0]] * clips
        placement = fc.assign_requests(pairs, world)
        clip_ids = [c for c in range(clips) if placement[c] == rank]
    # N>1 with the u8 exchange (NEXT-1, default): ranks produce u8 codes, the
    # gather moves 1176-byte rows, the encoder expands them to tokens
    u8x = world > 1 and args.exchange == "u8"
    # N>1 with the paper's column split (--exchange colsplit): every
    # rank keeps 1176/W columns of ALL rows (all-to-all of column blocks)
    colx = world > 1 and args.exchange == "colsplit"
    if colx and (clips != 1 or args.tokens != "f32"):
        raise SystemExit("--exchange colsplit: single-request configs, f32 tokens")
    # N>1 with the fused peer-store exchange (NEXT-1, --exchange p2p): every rank's
    # kernel writes its u8 codes straight into the encoder's buffer through a CUDA
    # IPC mapping (over NVLink), the exchange is one stream-ordered completion
    # collective, and the encoder expands the codes
    p2px = world > 1 and args.exchange == "p2p" and clips == 1
    if p2px:
        u8x = True
    if replicas:
        u8x = colx = p2px = False
    cfg = fc.ModelCfg(world_size=1 if replicas else world, sample_fps=wl.sample_fps,
                      token_dtype="u8" if u8x else args.tokens, color=args.color, surface_format=args.surface,
                      backend=args.backend)
    tok_bytes = 2 if args.tokens == "bf16" else 4
    plan0 = fc.Plan(meta, cfg)
    rp = plan0.rank(0 if replicas else rank)
    n_all = plan0.num_sampled * clips
    clips_all = clips
    if replicas:
        clips = len(clip_ids)  # this rank's clips
    # this rank's frames (global indices) -- only those are materialised
    my_frames = plan0.sampled_indices[rp["sampled_begin"]:rp["sampled_begin"] + rp["sampled_count"]]
    hosts = [synth.frames_nv12(wl, my_frames, "natural", clip=c) for c in clip_ids]
    if args.surface == "i420":  # the same samples as planar Y, U, V surfaces
        hosts = [{f: synth.nv12_to_i420(y, uv, wl.width, noise_seed=f) for f, (y, uv) in h.items()} for h in hosts]

    def stack_device(h):
        """One contiguous device stack per plane (Y, UV -- or Y, U, V for I420)
        per request (frames in index order); surfaces point into them."""
        fr = sorted(h)
        if not fr:
            return {}, None
        planes = tuple(torch.from_numpy(np.stack([h[f][p] for f in fr])).cuda() for p in range(len(h[fr[0]])))
        return {f: tuple(pl[i] for pl in planes) for i, f in enumerate(fr)}, planes

    stacks = [stack_device(h) for h in hosts]
    devs = [d for d, _ in stacks]
    surfs = [fc.SurfaceTable.from_tensors(d, wl.num_frames) for d in devs]
    rows = rp["row_end"] - rp["row_begin"]
    tdt = torch.bfloat16 if args.tokens == "bf16" else torch.float32
    xdt = torch.uint8 if u8x else tdt  # what the kernel writes and the gather moves
    outs = [torch.empty((world, max(rows, 1), 1176 // world) if colx else (max(rows, 1), 1176), dtype=xdt,
                        device="cuda") for _ in range(clips)]
    mines = [torch.empty((plan0.token_rows, 1176 // world), dtype=torch.float32, device="cuda") if colx else None
             for _ in range(clips)]
    comm = fc.NcclComm(rank, world) if world > 1 and not replicas else None
    xrank = 0 if replicas else rank  # the plan rank this process runs
    enc = cfg.encoder_rank
    fulls = [torch.empty((plan0.token_rows, 1176), dtype=xdt, device="cuda")
             if (world > 1 and rank == enc and not colx and not replicas) else None for _ in range(clips)]
    toks = [torch.empty((plan0.token_rows, 1176), dtype=tdt, device="cuda")
            if (u8x and rank == enc) else None for _ in range(clips)]
    peer = None
    if p2px:  # every rank's output = its rows of the encoder's code buffer (IPC-mapped off the encoder)
        hdl = [fc.ipc_export(fulls[0]) if rank == enc else None]
        dist.broadcast_object_list(hdl, src=enc)
        if rank == enc:
            outs[0] = fulls[0][rp["row_begin"]:rp["row_end"]]
        elif rows:
            peer = fc.PeerBuffer(hdl[0][0])
            outs[0] = peer.tensor((rows, 1176), torch.uint8, hdl[0][1] + rp["row_begin"] * 1176)
        done = torch.zeros(1, device="cuda")
    stream = torch.cuda.current_stream()

    def exchange(plans):
        """a10 (+ the encoder-side expand of the u8 exchange)."""
        if p2px:  # the codes are already in place: order the encoder after every rank's kernel
            dist.all_reduce(done)
            if rank == enc:
                fc.expand_tokens(plans[0], fulls[0], toks[0], args.tokens)
            return
        for pl, o, fl, tk, mn in zip(plans, outs, fulls, toks, mines):
            if colx:
                fc.scatter_columns(pl, rank, comm, o if rows else None, mn)
                continue
            fc.gather(pl, rank, comm, o if rows else None, fl)
            if tk is not None:
                fc.expand_tokens(pl, fl, tk, args.tokens)

    # one request per step on one rank: plan + launch in ONE C call (fc_submit;
    # small requests are bound by per-call host overhead)
    single = clips == 1 and not colx and not replicas and rows > 0

    def step(plans_keep, ev_a=None, ev_b=None):
        if single:
            if ev_a is not None:
                ev_a.record(stream)
            plans = [fc.submit(meta, cfg, xrank, surfs[0], outs[0])]   # a1-a4 + a5-a9
            plans_keep.append(plans)
            if ev_b is not None:
                ev_b.record(stream)
            if world > 1:
                exchange(plans)                        # a10
            if len(plans_keep) > 64:
                del plans_keep[0]  # one old plan per step (its work has long completed): no bursts
            return
        plans = [fc.Plan(meta, cfg) for _ in range(clips)]   # a1-a4 (host), one plan per request
        plans_keep.append(plans)
        if ev_a is not None:
            ev_a.record(stream)
        if rows and clips:
            if colx:
                fc.preprocess_colsplit(plans[0], rank, surfs[0], outs[0])  # a5-a9, column-block epilogue
            elif clips == 1 and not replicas:
                fc.preprocess(plans[0], xrank, surfs[0], outs[0])   # a5-a9 (one launch)
            else:  # a5-a9 for every request in ONE launch (same shape)
                fc.preprocess_batch([(pl, xrank, sf) for pl, sf in zip(plans, surfs)], outs)
        if ev_b is not None:
            ev_b.record(stream)
        if world > 1 and not replicas:
            exchange(plans)                        # a10
        if len(plans_keep) > 64:
            del plans_keep[:32]                   # older plans' work has long completed

    # host planning cost (a1-a4), timed separately; inside the
    # timed steps it overlaps the previous request's kernel
    tp0 = time.perf_counter()
    for _ in range(20):
        fc.Plan(meta, cfg)
    plan_us = (time.perf_counter() - tp0) / 20 * 1e6

    # L2 (126 MB on B200): a step whose own bytes (this rank's NV12 read + token
    # write) stay under 2x L2 could reuse cached inputs/outputs across steps, so
    # such steps are timed one by one with a 256 MB scratch write in between
    # (outside the events); larger steps stream through L2 on their own
    L2_BYTES = 126 * 2 ** 20
    my_step_bytes = clips * max(algorithmic_bytes(plan0, wl, plan0.rank(r), 1 if u8x else tok_bytes)
                                for r in ([xrank] if world > 1 and not replicas else [0]))
    if world == 1 or replicas:
        my_step_bytes = clips * algorithmic_bytes(plan0, wl, tok_bytes=tok_bytes)
    flush = my_step_bytes < 2 * L2_BYTES
    scratch = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device="cuda") if flush else None

    keep = []
    for _ in range(args.warmup):
        step(keep)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    sevs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]  # step boundaries
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = fc.lib().fc_kernel_launches()
    fevs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in range(args.steps)] if flush else None
    with ClockSampler(local) as clk:  # the headline pass: no per-step instrumentation
        torch.cuda.synchronize()
        if flush:  # cold L2 at every step: scratch write, then the step between its own events
            for k in range(args.steps):
                scratch.zero_()
                fevs[k][0].record(stream)
                step(keep)
                fevs[k][1].record(stream)
        else:
            t0.record(stream)
            for k in range(args.steps):
                step(keep)
            t1.record(stream)
        torch.cuda.synchronize()
    launches = fc.lib().fc_kernel_launches() - launches0
    if world > 1:
        dist.barrier()
    total_ms = sum(a.elapsed_time(b) for a, b in fevs) if flush else t0.elapsed_time(t1)
    # a second pass with per-step events (step boundaries, kernel launch) for
    # the median / min / kernel-time statistics
    torch.cuda.synchronize()
    for k in range(args.steps):
        sevs[k].record(stream)
        step(keep, *evs[k])
    sevs[args.steps].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    kern_ms = [a.elapsed_time(b) for a, b in evs] if (rows and clips) else [0.0]
    kern_avg = sum(kern_ms) / len(kern_ms)
    step_ms = [sevs[k].elapsed_time(sevs[k + 1]) for k in range(args.steps)]
    if os.environ.get("FC_BENCH_STEPS"):  # diagnostics: per-step kernel times
        print("kernel ms per step:", " ".join(f"{x:.3f}" for x in kern_ms), file=sys.stderr)
    # max over ranks
    stats = torch.tensor([total_ms, kern_avg, statistics.median(step_ms), min(step_ms), statistics.median(kern_ms),
                          min(kern_ms)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.MAX)
    total_ms, kern_max, step_med, step_min, kern_med, kern_min = stats.tolist()
    ms_per_step = total_ms / args.steps

    # CUDA-graph variant (one request on one GPU): fc_preprocess captured once
    # and replayed -- the same work without the per-call host path (plan reuse,
    # tensor maps in the kernel parameters; launches with more than 120 frames
    # upload a descriptor and are not captured)
    graph = None
    if world == 1 and clips == 1 and not replicas and not colx and rows and plan0.num_sampled > 120:
        graph = {"unavailable": "more than 120 frames per launch: the launch uploads a descriptor (not captured)"}
    elif world == 1 and clips == 1 and not replicas and not colx and rows:
        try:
            gs = torch.cuda.Stream()
            fc.preprocess(plan0, 0, surfs[0], outs[0], stream=gs)
            gs.synchronize()
            cg = torch.cuda.CUDAGraph()
            with torch.cuda.graph(cg, stream=gs):
                fc.preprocess(plan0, 0, surfs[0], outs[0], stream=gs)
            for _ in range(3):
                cg.replay()
            torch.cuda.synchronize()
            reps = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                    for _ in range(args.steps)]
            cur = torch.cuda.current_stream()
            ga, gb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ga.record(cur)
            for k in range(args.steps):
                if flush:
                    scratch.zero_()
                reps[k][0].record(cur)
                cg.replay()
                reps[k][1].record(cur)
            gb.record(cur)
            torch.cuda.synchronize()
            gms = (sum(a.elapsed_time(b) for a, b in reps) if flush else ga.elapsed_time(gb)) / args.steps
            graph = {"ms_per_step": round(gms, 4), "value": round(n_all / (gms * 1e-3), 2), "unit": "frames/s",
                     "note": "fc_preprocess captured once in a CUDA graph and replayed (same plan and surfaces)"}
            del cg
        except Exception as ex:  # noqa: BLE001 -- capture not possible for this launch
            graph = {"unavailable": str(ex)[:120]}

    # gather alone (N>1), timed separately for the NVLink report
    gather = None
    if world > 1 and not replicas:
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.barrier()
        torch.cuda.synchronize()
        g0.record(stream)
        for _ in range(max(3, args.steps // 4)):
            exchange([plan0] * clips)
        g1.record(stream)
        torch.cuda.synchronize()
        gms = torch.tensor([g0.elapsed_time(g1) / max(3, args.steps // 4)], dtype=torch.float64, device="cuda")
        dist.all_reduce(gms, op=dist.ReduceOp.MAX)
        gbytes = clips * sum((r["row_end"] - r["row_begin"]) * 1176 * (1 if u8x else tok_bytes)
                             for i, r in enumerate(plan0.ranks()) if i != enc)
        if colx:  # bytes into the busiest rank: every other rank's rows x its C columns
            gbytes = max((plan0.token_rows - (r["row_end"] - r["row_begin"])) * (1176 // world) * 4
                         for r in plan0.ranks())
        if p2px:  # the bytes crossed NVLink inside the ranks' kernels; this times completion + expand
            gbytes = sum((r["row_end"] - r["row_begin"]) * 1176 for i, r in enumerate(plan0.ranks()) if i != enc)
        gather = {"exchange": "fused peer stores of u8 codes (IPC) + completion all-reduce + encoder expand" if p2px
                  else "column split all-to-all (P:527-530)" if colx else
                  "u8 codes + encoder expand" if u8x else args.tokens,
                  "ms": round(gms.item(), 4), "bytes_into_encoder": gbytes,
                  "GB/s": round(gbytes / (gms.item() * 1e-3) / 1e9, 1), "nvlink_nominal_GB/s": 900,
                  "nvlink_measured_peer_GB/s": 770}

    # e2e: the same step from pinned host NV12 through the public API.  Each
    # step uploads its request's frames (visible bytes only: 2-D copies of W
    # bytes per row) on a copy stream into one of two device surface sets, so
    # request k+1 uploads while request k computes; the result's first token
    # row per request comes back to the host.  Timed from the first upload to
    # the last read-back.
    from cuda.bindings import runtime as cudart

    pinned = [tuple(torch.from_numpy(np.stack([h[f][p] for f in sorted(h)])).pin_memory()
                    for p in range(len(next(iter(h.values()))))) if h else None for h in hosts]
    stacks2 = [stack_device(h) for h in hosts]
    surfs2 = [fc.SurfaceTable.from_tensors(d, wl.num_frames) for d, _ in stacks2]
    sets = [([st for _, st in stacks], surfs), ([st for _, st in stacks2], surfs2)]
    res_host = torch.empty((clips, 1176), dtype=tdt).pin_memory()
    W, H = wl.width, wl.height
    h2d = sum(len(h) * (W * H + W * (H // 2)) for h in hosts)  # NV12 and I420 carry the same bytes
    widths = (W, W // 2, W // 2) if args.surface == "i420" else (W, W)  # visible bytes per plane row
    e2e_steps = max(3, min(args.steps, 10))
    cstream = torch.cuda.Stream()
    up_done = [torch.cuda.Event(), torch.cuda.Event()]
    used = [torch.cuda.Event(), torch.cuda.Event()]
    H2D = cudart.cudaMemcpyKind.cudaMemcpyHostToDevice

    def upload(k):
        dv_set = sets[k & 1][0]
        cstream.wait_event(used[k & 1])  # the compute of request k-2 released this set
        for pc, st in zip(pinned, dv_set):
            if pc is None:
                continue
            for src, dst, wb in zip(pc, st, widths):  # one 2-D copy per plane stack (visible bytes per row)
                err, = cudart.cudaMemcpy2DAsync(dst.data_ptr(), dst.stride(1), src.data_ptr(), src.stride(1), wb,
                                                src.shape[0] * src.shape[1], H2D, cstream.cuda_stream)
                assert err == cudart.cudaError_t.cudaSuccess, err
        up_done[k & 1].record(cstream)

    def e2e_step(k, keep):
        sf_set = sets[k & 1][1]
        stream.wait_event(up_done[k & 1])
        if single:
            plans = [fc.submit(meta, cfg, xrank, sf_set[0], outs[0])]
        else:
            plans = [fc.Plan(meta, cfg) for _ in range(clips)]
        keep.append(plans)
        if rows and clips and not single:
            if colx:
                fc.preprocess_colsplit(plans[0], rank, sf_set[0], outs[0])
            elif clips == 1 and not replicas:
                fc.preprocess(plans[0], xrank, sf_set[0], outs[0])
            else:
                fc.preprocess_batch([(pl, xrank, sf) for pl, sf in zip(plans, sf_set)], outs)
        used[k & 1].record(stream)
        if world > 1 and not replicas:
            exchange(plans)
        if colx:  # the first row of this rank's column slice
            res_host[0][:1176 // world].copy_(mines[0][0], non_blocking=True)
        elif world == 1 or replicas or rank == enc:  # one token row of every request's result back to the host
            for c in range(clips):
                src = (toks[c] if u8x else fulls[c]) if (world > 1 and not replicas) else outs[c]
                res_host[c].copy_(src[0], non_blocking=True)

    for k in range(2):  # warm-up of both surface sets
        upload(k)
        e2e_step(k, keep)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    cstream.wait_event(e0)
    upload(0)
    for k in range(e2e_steps):
        if k + 1 < e2e_steps:
            upload(k + 1)  # overlaps request k's compute
        e2e_step(k, keep)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([e0.elapsed_time(e1) / e2e_steps], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_ms = e2e_ms.item()

    # e2e with the FULL result read back to the host every step (host -> host;
    # the default e2e keeps the tokens on the GPU for the encoder and reads one
    # row back).  Only where the result fits a 2 GiB pinned buffer.
    full_rb = None
    results = []
    if colx:
        results = [mines[0]]
    elif world == 1 or replicas:
        results = outs[:clips]
    elif rank == enc:
        results = [(toks[c] if u8x else fulls[c]) for c in range(clips)]
    rb_bytes = sum(r.numel() * r.element_size() for r in results)
    # the same decision on every rank (the exchange inside e2e_step is collective)
    if clips_all * plan0.token_rows * 1176 * tok_bytes <= (2 << 30):
        rb_host = [torch.empty(r.shape, dtype=r.dtype).pin_memory() for r in results]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        cstream.wait_event(f0)
        upload(0)
        for k in range(3):
            if k + 1 < 3:
                upload(k + 1)
            e2e_step(k, keep)
            for hst, r in zip(rb_host, results):
                hst.copy_(r, non_blocking=True)
        f1.record(stream)
        torch.cuda.synchronize()
        frb = torch.tensor([f0.elapsed_time(f1) / 3], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(frb, op=dist.ReduceOp.MAX)
        full_rb = {"value": round(n_all / (frb.item() * 1e-3), 2), "unit": "frames/s",
                   "ms_per_step": round(frb.item(), 3), "h2d_bytes_per_step": None,
                   "d2h_bytes_per_step": rb_bytes}

    if rank == 0:
        peak, peak_kind = load_peaks()
        if world == 1:
            abytes = clips * algorithmic_bytes(plan0, wl, tok_bytes=tok_bytes)
            kern_for_roof = kern_avg
        else:  # dominant kernel = this rank's launch; bytes of the largest shard
            abytes = clips * max(algorithmic_bytes(plan0, wl, r, 1 if u8x else tok_bytes) for r in plan0.ranks())
            kern_for_roof = kern_max
        achieved = abytes / (kern_for_roof * 1e-3) / 1e9
        same_kernel = (world == 1 and args.tokens == "f32" and args.color == "bt601" and args.surface == "nv12"
                       and args.backend == "pil")
        traffic = load_traffic(args.config) if same_kernel else None
        # second roofline: the kernel is bound by instruction issue;
        # warp instructions per launch from the committed ncu capture of this config
        winstr = load_traffic(args.config, "warp_instructions_per_launch") if same_kernel else None
        issue = None
        if winstr:
            clk_mhz = clk.summary().get("sm_mhz") or 1965
            peak_g = 148 * 4 * clk_mhz * 1e6 / 1e9  # warp instructions per second (G), 4 schedulers/SM
            ach_g = winstr / (kern_for_roof * 1e-3) / 1e9
            issue = {"bound": "issue", "achieved": round(ach_g, 1), "peak": round(peak_g, 1),
                     "unit": "G warp-instr/s", "frac": round(ach_g / peak_g, 4),
                     "warp_instructions_per_launch": int(winstr)}
        line = {
            "metric": METRIC, "value": round(n_all / (ms_per_step * 1e-3), 2), "unit": "frames/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": f"u8->{args.tokens}",
            "data": "synthetic",
            "config": {"workload": f"{args.config}: {wl.note}", "frames": n_all, "requests": clips,
                       "resized_hw": list(plan0.resized), "grid_thw": list(plan0.grid_thw),
                       "token_bytes": clips_all * plan0.token_rows * 1176 * tok_bytes,
                       "parallelism": (f"replicas{world} (whole clips, LPT)" if replicas else f"gop-dp{world}"),
                       "color": args.color, "surface": args.surface, "backend": args.backend,
                       "l2": (f"L2 flushed between timed steps (256 MB scratch write outside the step events): "
                              f"{my_step_bytes / 1e6:.0f} MB per step < 2x the 126 MB L2" if flush else
                              f"per-step inputs+outputs ({my_step_bytes / 1e9:.2f} GB) exceed the 126 MB L2; no flush"),
                       "kernel_ms_avg": round(kern_max if world > 1 else kern_avg, 4)},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic, "peak_kind": peak_kind,
                         "algorithmic_bytes_per_launch": abytes, **({"issue": issue} if issue else {})},
            "step_ms": {"mean": round(ms_per_step, 4), "median": round(step_med, 4), "min": round(step_min, 4),
                        "kernel_mean": round(kern_max if world > 1 else kern_avg, 4),
                        "kernel_median": round(kern_med, 4), "kernel_min": round(kern_min, 4),
                        "note": "second pass with per-step CUDA events on the launching stream; max over ranks"},
            "preprocess_ms_max_over_ranks": round(kern_max if world > 1 else kern_avg, 4),
            "plan_host_us": round(plan_us, 1),
            "gpu_launches": int(launches),  # fc_kernel_launches() delta over the timed region (this rank)
            "e2e": {"value": round(n_all / (e2e_ms * 1e-3), 2), "unit": "frames/s", "ms_per_step": round(e2e_ms, 3),
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 1176 * tok_bytes * clips},
            "clocks": clk.summary(),
        }
        if gather is not None:
            line["gather"] = gather
        if graph is not None:
            line["cuda_graph"] = graph
        if full_rb is not None:  # the same e2e with the whole token tensor read back (host -> host)
            full_rb["h2d_bytes_per_step"] = h2d
            line["e2e_full_readback"] = full_rb
        if world == 1 and not args.no_cpu_baseline:
            cores = len(os.sched_getaffinity(0))
            pairs = min(plan0.grid_thw[0], 60)
            dt, f = oracle_sample(wl, pairs, cores, args.color, args.backend)
            dt1, f1 = oracle_sample(wl, 1, 1, args.color, args.backend)  # one temporal pair on one core
            line["cpu_baseline"] = {"value": round(f / dt, 3), "unit": "frames/s", "cores": cores,
                                    "kind": "oracle",
                                    "sample": f"{f} sampled frames ({pairs} temporal pairs) of {args.config}, "
                                              f"natural content, {dt:.1f} s wall on {cores} threads",
                                    "single_core": {"value": round(f1 / dt1, 3), "unit": "frames/s", "cores": 1,
                                                    "sample": f"{f1} sampled frames (1 temporal pair), {dt1:.2f} s"}}
        print(json.dumps(line), flush=True)
    if peer is not None:
        peer.close()
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(synth.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--tokens", default="f32", choices=["f32", "bf16"],
                    help="token dtype (NEXT-4 variant; the BASELINE metric is f32)")
    ap.add_argument("--exchange", default="u8", choices=["u8", "f32", "colsplit", "p2p"],
                    help="N>1 exchange: u8 codes + encoder-side expand (default), the tokens themselves, the "
                         "paper's column split (every rank keeps 1176/N columns of all rows), or fused peer stores "
                         "(each rank's kernel writes its codes into the encoder's buffer over NVLink)")
    ap.add_argument("--color", default="bt601", choices=["bt601", "bt709", "bt601_full", "bt709_full"],
                    help="YUV->RGB matrix (NEXT-4 variant; the BASELINE metric is bt601)")
    ap.add_argument("--backend", default="pil", choices=["pil", "torchvision"],
                    help="HF processor arithmetic (DESIGN.md R21): Pillow bicubic + HF normalise, or torch's "
                         "uint8 antialiased bicubic + the fused normalisation (same kernel, other tables)")
    ap.add_argument("--surface", default="nv12", choices=["nv12", "i420"],
                    help="decoded surface layout: NV12 (interleaved chroma) or I420 (planar U, V)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
