"""Seeded synthetic inputs for the FlashCodec preprocessing path.

This module holds NO arithmetic of the method (no sampling, resize, colour or
layout code).  It only describes the paper-shaped workloads of
BASELINE.json's configs and draws deterministic NV12 frame content.  Both the
product tests/bench and the oracle checks consume it.

Workloads (BASELINE.json configs):
  c1  4 s 320x240 @30, 1 GOP, 2 fps sampling
  c2  60 s 1920x1080 @30, GOP 30, 2 fps
  c3  10 min 1280x720 @30, 256 GOPs (80x71 + 176x70 frames), 1 fps
  c4  30 s 3840x2160 @30, GOP 30, 2 fps
  c5  64 clips of 10 s 854x480 @30, GOP 30, 2 fps (throughput mode)

Content kinds (seed = 1000 + config id, per-frame content depends on the
frame index so that sampling mistakes change the tokens):
  natural  limited-range smooth fields + integer noise (timed runs)
  uniform  Y, U, V uniform over [0, 255] (clamps, bicubic overshoot)
  edges    16-px checkerboards, Y in {16, 235}, saturated chroma (ringing)
Surfaces use an NVDEC-like pitch, round_up(width, 256).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    width: int
    height: int
    num_frames: int
    fps: tuple[int, int]
    gop_sizes: tuple[int, ...]
    sample_fps: float
    clips: int = 1
    note: str = ""

    @property
    def gop_start(self) -> list[int]:
        out, s = [], 0
        for g in self.gop_sizes:
            out.append(s)
            s += g
        return out

    @property
    def pitch(self) -> int:
        return pitch_for(self.width)

    @property
    def seed(self) -> int:
        return 1000 + int(self.name[1:]) if self.name[1:].isdigit() else 999


def pitch_for(width: int) -> int:
    return (width + 255) // 256 * 256


CONFIGS = {
    "c1": Workload("c1", 320, 240, 120, (30, 1), (120,), 2.0,
                   note="4 s 320x240 synthetic NV12 video, 2 fps, single GOP, 1 GPU"),
    "c2": Workload("c2", 1920, 1080, 1800, (30, 1), (30,) * 60, 2.0,
                   note="60 s 1080p30, 2 fps, Qwen2.5-VL max_pixels, GOP=30"),
    "c3": Workload("c3", 1280, 720, 18000, (30, 1), (71,) * 80 + (70,) * 176, 1.0,
                   note="10 min 720p30, 1 fps, 256 GOPs"),
    "c4": Workload("c4", 3840, 2160, 900, (30, 1), (30,) * 30, 2.0,
                   note="30 s 4K30, 2 fps, heavy resize"),
    "c5": Workload("c5", 854, 480, 300, (30, 1), (30,) * 10, 2.0, clips=64,
                   note="64 concurrent 10 s 480p clips (throughput mode)"),
}


def frame_nv12(width: int, height: int, frame: int, kind: str = "natural", seed: int = 0,
               pitch: int | None = None) -> tuple[np.ndarray, np.ndarray]:
    """One NV12 frame: (y [H, pitch] u8, uv [H/2, pitch] u8 interleaved U,V).
    Bytes in the pitch padding are filled with noise (they must never matter)."""
    pitch = pitch or pitch_for(width)
    rng = np.random.default_rng([seed, frame, {"natural": 1, "uniform": 2, "edges": 3}[kind]])
    y = rng.integers(0, 256, size=(height, pitch), dtype=np.uint8)
    uv = rng.integers(0, 256, size=(height // 2, pitch), dtype=np.uint8)
    if kind == "uniform":
        return y, uv
    if kind == "natural":
        ph = rng.random(6) * 2 * np.pi
        xs = np.arange(width, dtype=np.float32)
        ys = np.arange(height, dtype=np.float32)
        fx = np.sin(xs * (2 * np.pi / (37.0 + 11 * (frame % 5))) + ph[0]).astype(np.float32)
        fy = np.sin(ys * (2 * np.pi / (53.0 + 7 * (frame % 3))) + ph[1]).astype(np.float32)
        base = 125.0 + 50.0 * fx[None, :] + 40.0 * fy[:, None]
        noise = rng.integers(-6, 7, size=(height, width), dtype=np.int16)
        y[:, :width] = np.clip(base + noise, 16, 235).astype(np.uint8)
        cx = np.arange(width // 2, dtype=np.float32)
        cy = np.arange(height // 2, dtype=np.float32)
        u = 128 + 60 * np.sin(cx * (2 * np.pi / 71.0) + ph[2])[None, :] + 20 * np.sin(cy * (2 * np.pi / 41.0) + ph[3])[:, None]
        v = 128 + 55 * np.sin(cx * (2 * np.pi / 59.0) + ph[4])[None, :] + 25 * np.sin(cy * (2 * np.pi / 47.0) + ph[5])[:, None]
        uvv = uv[:, : width].reshape(height // 2, width // 2, 2)
        uvv[..., 0] = np.clip(u, 16, 240).astype(np.uint8)
        uvv[..., 1] = np.clip(v, 16, 240).astype(np.uint8)
        return y, uv
    if kind == "edges":
        sh = frame % 16
        xs = (np.arange(width) + sh) // 16
        ys = (np.arange(height) + 3 * sh) // 16
        chk = (xs[None, :] + ys[:, None]) % 2
        y[:, :width] = np.where(chk == 1, 235, 16).astype(np.uint8)
        cxs = (np.arange(width // 2) + sh) // 8
        cys = (np.arange(height // 2) + sh) // 8
        cchk = (cxs[None, :] + cys[:, None]) % 2
        uvv = uv[:, : width].reshape(height // 2, width // 2, 2)
        uvv[..., 0] = np.where(cchk == 1, 240, 16).astype(np.uint8)
        uvv[..., 1] = np.where(cchk == 1, 16, 240).astype(np.uint8)
        return y, uv
    raise ValueError(kind)


def frames_nv12(wl: Workload, indices, kind: str = "natural", clip: int = 0) -> dict:
    """Materialise only the listed frames of workload `wl` (clip `clip`)."""
    seed = wl.seed * 1000 + clip
    return {int(i): frame_nv12(wl.width, wl.height, int(i), kind, seed, wl.pitch) for i in indices}


def nv12_to_i420(y: np.ndarray, uv: np.ndarray, width: int, pitch_c: int | None = None, noise_seed: int = 0):
    """The same samples as planar I420: (y, u, v) with U = the even bytes and
    V = the odd bytes of the interleaved chroma rows (data movement only).  The
    chroma planes get pitch `pitch_c` (default pitch_for(width/2)) with noise in
    the padding, which must never matter."""
    cw = width // 2
    pc = pitch_c or pitch_for(cw)
    rng = np.random.default_rng(noise_seed)
    u = rng.integers(0, 256, (uv.shape[0], pc), dtype=np.uint8)
    v = rng.integers(0, 256, (uv.shape[0], pc), dtype=np.uint8)
    u[:, :cw] = uv[:, 0:2 * cw:2]
    v[:, :cw] = uv[:, 1:2 * cw:2]
    return y, u, v


def to_device(frames: dict, device="cuda") -> dict:
    """Host planes -> device tensors; works for NV12 (y, uv) and I420 (y, u, v) tuples."""
    import torch
    return {k: tuple(torch.from_numpy(p).to(device) for p in planes) for k, planes in frames.items()}
