"""Seeded synthetic gradient generators shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the aggregation method (no medians, sums,
distances or selections); it only draws the input matrices.  Both sides of a
parity test receive the *same bits*: the matrix is drawn once (on CPU or on a
CUDA device) and copied to the other side.

Recipe:

* honest rows (n - f of them):  x_i = mu + sigma * z_i,  mu ~ N(0, 0.01^2) per
  coordinate (fixed per seed), sigma = 0.01, z_i ~ N(0, 1);
* Byzantine rows (f of them, at seeded positions), the paper's two attacks
  (§5.4 "random values" and "reversed vector x(-100)"):
  ceil(f/2) rows  -100 * (mu + sigma * z_b)  and  floor(f/2) rows  N(0, 1);
* ``kind="clean"``: all n rows honest;
* ``kind="separated"``: as "byzantine", but honest row spreads follow a seeded
  permutation of the ladder sigma_j = sigma * 1.04^j, so every Krum score (and
  every Bulyan round's best score) is separated from the next by far more than
  the 1e-4 relative gap of SURVEY.md §8c-6: the selection is then well posed and
  the GPU must reproduce it exactly (tests/gpu_helpers.py).

Shapes follow PAPER.md Table 1 (l.481-498) and BASELINE.json ``configs``.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np
import torch

BASE_SEED = 20105888

# BASELINE.json configs; d values per SURVEY.md §8 (C1..C5).
MNIST_CNN_D = 79_510          # PAPER.md l.489 (Table 1)
CIFARNET_D = 1_756_426        # PAPER.md l.490 (Table 1)
RESNET50_D = 25_557_032       # torchvision ResNet-50 (BASELINE.json "~25.6M")
VGG16_D = 138_357_544         # torchvision VGG16 (BASELINE.json "~138M")


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    n: int
    f: int
    d: int
    rules: tuple


CONFIGS = {
    "C1": Config("C1-mnist", 11, 2, MNIST_CNN_D, ("median", "krum", "bulyan", "trimmed_mean", "average", "multi_krum")),
    "C2": Config("C2-cifarnet", 19, 4, CIFARNET_D, ("average", "median", "trimmed_mean", "krum", "multi_krum", "bulyan")),
    "C3": Config("C3-resnet50", 31, 7, RESNET50_D, ("bulyan", "multi_krum")),
    "C4": Config("C4-vgg16", 31, 7, VGG16_D, ("median", "krum")),
}


def sweep_config(n: int, d: int = RESNET50_D) -> Config:
    """C5: n = 4f + 3, f = (n - 3) / 4 (f = floor((n-3)/4))."""
    return Config(f"C5-n{n}", n, (n - 3) // 4, d,
                  ("average", "median", "trimmed_mean", "krum", "multi_krum", "bulyan"))


def aligned_ld(d: int) -> int:
    """Row pitch (in floats) that keeps every row 16-byte aligned."""
    return (d + 3) // 4 * 4


def byzantine_positions(n: int, f: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed ^ 0x5EED)
    return np.sort(rng.permutation(n)[:f])


def make_gradients(n: int, f: int, d: int, seed: int, kind: str = "byzantine",
                   device="cpu", ld: int | None = None) -> torch.Tensor:
    """Return an fp32 tensor of shape [n, ld] (ld >= d, columns >= d are zero).

    Rows are the n worker gradients; ``[:, :d]`` is the data.  Generated with a
    torch.Generator on ``device`` so large matrices never touch the host.
    """
    if kind not in ("byzantine", "clean", "separated"):
        raise ValueError(kind)
    ld = aligned_ld(d) if ld is None else ld
    dev = torch.device(device)
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    x = torch.zeros((n, ld), dtype=torch.float32, device=dev)
    mu = torch.randn(d, generator=g, device=dev, dtype=torch.float32).mul_(0.01)
    byz = set(byzantine_positions(n, f, seed).tolist()) if kind != "clean" else set()
    ladder = None
    if kind == "separated":
        rank = np.random.default_rng(seed ^ 0x1ADD).permutation(n)
        ladder = [float(1.04 ** int(r)) for r in rank]
    n_rev = math.ceil(len(byz) / 2)
    byz_sorted = sorted(byz)
    reversed_rows = set(byz_sorted[:n_rev])
    for i in range(n):
        row = x[i, :d]
        if i in byz and i not in reversed_rows:
            row.copy_(torch.randn(d, generator=g, device=dev, dtype=torch.float32))
        else:
            torch.randn(d, generator=g, device=dev, dtype=torch.float32, out=row)
            row.mul_(0.01 if ladder is None else 0.01 * ladder[i]).add_(mu)
            if i in reversed_rows:
                row.mul_(-100.0)
    return x


def to_bf16(x: torch.Tensor) -> torch.Tensor:
    """bf16 copy of a generated fp32 matrix (torch's round-to-nearest-even
    conversion), for the bf16-input variant.  Input generation
    only: both sides receive these bf16 bits.  A 2-D matrix keeps 16-byte
    aligned rows: its row length is padded with zeros to a multiple of 8."""
    if x.dim() == 2 and x.shape[1] % 8:
        y = torch.zeros((x.shape[0], (x.shape[1] + 7) // 8 * 8), dtype=torch.bfloat16, device=x.device)
        y[:, : x.shape[1]] = x
        return y
    return x.to(torch.bfloat16)


def bf16_bits(x: torch.Tensor) -> np.ndarray:
    """The uint16 bit patterns of a bf16 tensor (what the oracle takes)."""
    return x.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)


def make_sharded_gradients(n: int, f: int, d: int, seed: int, rank: int, world: int,
                           device="cpu", kind: str = "byzantine") -> tuple[torch.Tensor, int, int]:
    """d-sharded view for rank ``rank``: rows restricted to its coordinate slice.

    Slice boundaries are multiples of 1024 coordinates.  Each
    rank draws its own slice from a per-slice seed, so the union over ranks is
    a fixed matrix for a given (seed, world).  Returns (x_local, lo, hi).
    """
    lo, hi = shard_bounds(d, rank, world)
    x = make_gradients(n, f, hi - lo, seed * 1000 + rank * 7 + world, kind=kind, device=device)
    return x, lo, hi


def shard_bounds(d: int, rank: int, world: int) -> tuple[int, int]:
    per = (d + world - 1) // world
    per = (per + 1023) // 1024 * 1024
    lo = min(d, rank * per)
    hi = min(d, lo + per)
    return lo, hi


def adversarial_rows(n: int, d: int, seed: int) -> np.ndarray:
    """Small-d adversarial matrix: NaN/Inf/-0 payloads, exact duplicates and
    values crafted for ties.  Returns float32 [n, d]."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, d)).astype(np.float32) * np.float32(0.01)
    if n >= 4:
        x[1] = x[0]                                   # exact duplicate row
    specials = np.array([np.nan, np.inf, -np.inf, -0.0, 0.0, 1e30, -1e30,
                         np.float32(1.4e-45), -np.float32(1.4e-45)], dtype=np.float32)
    mask = rng.random((n, d)) < 0.08
    x[mask] = rng.choice(specials, size=int(mask.sum()))
    # columns of identical values (ties everywhere) and symmetric pairs
    if d >= 3:
        x[:, 0] = np.float32(0.25)
        x[:, 1] = np.where(np.arange(n) % 2 == 0, np.float32(1.0), np.float32(-1.0))
        x[:, 2] = -0.0
    if d >= 4:
        x[:, 3] = np.where(np.arange(n) % 3 == 0, np.float32(0.0), np.float32(-0.0))   # mixed-sign zeros
    return x
