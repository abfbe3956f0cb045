"""The reference's benchmark harness (bench.hpp:49-501) driving the B200 engine.

Same configuration keys (``BenchConfig``, unknown keys rejected, bench.hpp:83-127), same record
schema (``BenchRecord``: the pinned 23-column CSV header and JSON object, bench.hpp:189-297) and
the same input stream (``make_problem``: per slot q, k, v, d_out from one mt19937_64(seed),
bench.hpp:320-337), so GPU rows and the reference's CPU rows share a schema and their counter
columns agree exactly. Timing: each run times ``forward_all`` then ``backward_all`` over every
batch x head slot (bench.hpp:372-387) — here one launch each over all slots, timed with CUDA
events on the launching stream; ``prepro_ms`` is the GPU preprocessor (plus RCM and the device
mask permutation for "+rcm" rows, bench.hpp:448-455).

``precision`` keeps the reference's vocabulary; the engine computes in bf16 with fp32
accumulation whatever it says (documented in DESIGN.md). ``verify`` compares the forward output
with a plain fp32 PyTorch masked softmax attention on the same device (the harness's checker, like
the reference's naive_forward; it is not the engine).
"""
from __future__ import annotations

import ctypes as C
import json
import math
import statistics
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np

from . import _lib
from .blockmask import (BlockSpec, EngineCounters, Variant, attn_bwd_device, attn_fwd_device, bandwidth,
                        generate, parse_variant, permute_mask, permute_rows, preprocess_mask, rcm_order, to_string)

CSV_HEADER = ("variant,mask,n,block_i,block_j,batch,heads,runs,precision,prepro_ms,fwd_ms_mean,"
              "fwd_ms_std,bwd_ms_mean,bwd_ms_std,total_ms_mean,blocks_visited,blocks_processed,"
              "mask_block_reads,skipped_by_binblk,skipped_mask_reads_by_run,block_density,"
              "element_density,max_abs_err_vs_oracle")

PRECISIONS = ("single", "double")


def fmt_double(v: float) -> str:
    """std::setprecision(17) << v (bench.hpp:179-183): %.17g without trailing-zero padding."""
    s = "%.17g" % v
    if "e" in s:
        mant, exp = s.split("e")
        sign = exp[0]
        digits = exp[1:].lstrip("0").rjust(2, "0")
        s = f"{mant}e{sign}{digits}"
    return s


@dataclass
class BenchConfig:
    """bench.hpp:49-151."""
    mask_spec: str = "causal"
    seq_lengths: List[int] = field(default_factory=lambda: [1024])
    block_i: int = 64
    block_j: int = 64
    variants: List[Variant] = field(default_factory=lambda: list(Variant))
    batch: int = 4
    heads: int = 32
    runs: int = 100
    warmup: int = 5
    head_dim: int = 64
    precision: str = "double"
    rcm: bool = False
    verify: bool = False
    seed: int = 1
    oracle_limit: int = 2048
    memory_limit_gb: float = 4.0
    threads: int = 1

    KEYS = ("mask_spec", "seq_lengths", "block_i", "block_j", "variants", "batch", "heads", "runs",
            "warmup", "head_dim", "precision", "rcm", "verify", "seed", "oracle_limit",
            "memory_limit_gb", "threads")

    def validate(self) -> None:
        BlockSpec(self.block_i, self.block_j).validate()
        if self.runs < 1:
            raise ValueError("runs must be >= 1")
        if self.batch < 1 or self.heads < 1:
            raise ValueError("batch and heads must be >= 1")
        if self.head_dim < 1:
            raise ValueError("head_dim must be >= 1")
        if not self.variants:
            raise ValueError("need at least one variant")
        if self.threads < 1:
            raise ValueError("threads must be >= 1")
        if not self.memory_limit_gb > 0.0:
            raise ValueError("memory limit must be positive")
        if not self.seq_lengths:
            raise ValueError("seq_lengths must be non-empty")
        if self.precision not in PRECISIONS:
            raise ValueError(f"unknown precision: '{self.precision}' (expected single, double)")

    @staticmethod
    def from_json(obj) -> "BenchConfig":
        if isinstance(obj, str):
            obj = json.loads(obj)
        c = BenchConfig()
        for key, val in obj.items():
            if key not in BenchConfig.KEYS:
                raise ValueError(f"unknown config key: '{key}'")
            if key == "variants":
                val = [parse_variant(v) for v in val]
            setattr(c, key, val)
        c.validate()
        return c

    def to_json(self) -> dict:
        d = {k: getattr(self, k) for k in self.KEYS}
        d["variants"] = [to_string(v) for v in self.variants]
        return d


@dataclass
class BenchRecord:
    """bench.hpp:189-297: one row per (mask, length, variant)."""
    variant: Variant = Variant.dense
    mask: str = ""
    n: int = 0
    block_i: int = 0
    block_j: int = 0
    batch: int = 0
    heads: int = 0
    runs: int = 0
    precision: str = "double"
    prepro_ms: float = 0.0
    fwd_ms_mean: float = 0.0
    fwd_ms_std: float = 0.0
    bwd_ms_mean: float = 0.0
    bwd_ms_std: float = 0.0
    total_ms_mean: float = 0.0
    counters: EngineCounters = field(default_factory=EngineCounters)
    block_density: float = 0.0
    element_density: float = 0.0
    max_abs_err_vs_oracle: Optional[float] = None
    bandwidth_before: Optional[int] = None
    bandwidth_after: Optional[int] = None

    def csv_row(self) -> str:
        c = self.counters
        f = [to_string(self.variant), self.mask, str(self.n), str(self.block_i), str(self.block_j),
             str(self.batch), str(self.heads), str(self.runs), self.precision, fmt_double(self.prepro_ms),
             fmt_double(self.fwd_ms_mean), fmt_double(self.fwd_ms_std), fmt_double(self.bwd_ms_mean),
             fmt_double(self.bwd_ms_std), fmt_double(self.total_ms_mean), str(c.blocks_visited),
             str(c.blocks_processed), str(c.mask_block_reads), str(c.skipped_by_binblk),
             str(c.skipped_mask_reads_by_run), fmt_double(self.block_density),
             fmt_double(self.element_density),
             "" if self.max_abs_err_vs_oracle is None else fmt_double(self.max_abs_err_vs_oracle)]
        return ",".join(f)

    @staticmethod
    def parse_csv_row(line: str) -> "BenchRecord":
        f = line.split(",")
        if len(f) != 23:
            raise ValueError(f"expected 23 CSV fields, got {len(f)}")
        if f[8] not in PRECISIONS:
            raise ValueError(f"unknown precision: '{f[8]}' (expected single, double)")
        return BenchRecord(
            parse_variant(f[0]), f[1], int(f[2]), int(f[3]), int(f[4]), int(f[5]), int(f[6]), int(f[7]), f[8],
            float(f[9]), float(f[10]), float(f[11]), float(f[12]), float(f[13]), float(f[14]),
            EngineCounters(int(f[15]), int(f[16]), int(f[17]), int(f[18]), int(f[19])), float(f[20]),
            float(f[21]), float(f[22]) if f[22] else None)

    def to_json(self) -> dict:
        c = self.counters
        j = {"variant": to_string(self.variant), "mask": self.mask, "n": self.n, "block_i": self.block_i,
             "block_j": self.block_j, "batch": self.batch, "heads": self.heads, "runs": self.runs,
             "precision": self.precision, "prepro_ms": self.prepro_ms, "fwd_ms_mean": self.fwd_ms_mean,
             "fwd_ms_std": self.fwd_ms_std, "bwd_ms_mean": self.bwd_ms_mean, "bwd_ms_std": self.bwd_ms_std,
             "total_ms_mean": self.total_ms_mean, "blocks_visited": c.blocks_visited,
             "blocks_processed": c.blocks_processed, "mask_block_reads": c.mask_block_reads,
             "skipped_by_binblk": c.skipped_by_binblk, "skipped_mask_reads_by_run": c.skipped_mask_reads_by_run,
             "block_density": self.block_density, "element_density": self.element_density}
        if self.max_abs_err_vs_oracle is not None:
            j["max_abs_err_vs_oracle"] = self.max_abs_err_vs_oracle
        if self.bandwidth_before is not None:
            j["bandwidth_before"] = self.bandwidth_before
        if self.bandwidth_after is not None:
            j["bandwidth_after"] = self.bandwidth_after
        return j


def make_problem(seed: int, slots: int, n: int, d: int):
    """bench.hpp:320-337 through libbbm's mt19937_64 (bit-identical to the reference's stream):
    float arrays q, k, v, d_out of shape [slots][n][d]."""
    arrs = [np.empty((slots, n, d), np.float32) for _ in range(4)]
    _lib.check(_lib.lib.bbm_make_problem(seed, slots, n, d, *[_lib.ptr(a, C.c_float) for a in arrs]))
    return tuple(arrs)


def estimated_gb(n: int, head_dim: int, slots: int, precision: str) -> float:
    """bench.hpp:303-311 (the reference's guard, kept so configs are refused identically)."""
    es = 4.0 if precision == "single" else 8.0
    nd = float(n) * float(head_dim)
    b = slots * (5.0 * nd * es + 2.0 * n * 8.0) + 8.0 * nd * 8.0 + n * ((n + 63) // 64) * 8.0
    return b / (1024.0 ** 3)


def _torch_reference_forward(q, k, v, scale, dense_mask):
    """fp32 masked softmax attention with plain PyTorch ops (the harness's checker)."""
    import torch

    s = torch.einsum("snd,smd->snm", q.float(), k.float()) * scale
    if dense_mask is not None:
        s = s.masked_fill(~dense_mask, float("-inf"))
    m = s.amax(-1, keepdim=True)
    p = torch.where(torch.isinf(m), torch.zeros_like(s), torch.exp(s - m))
    l = p.sum(-1, keepdim=True)
    o = torch.einsum("snm,smd->snd", p, v.float())
    return torch.where(l > 0, o / l.clamp_min(1e-30), torch.zeros_like(o))


def _bench_variant(cfg, tensors, mask, prep, prepro_ms, variant, label, dev):
    import torch

    q, k, v, g = tensors
    slots, n, d = q.shape
    scale = 1.0 / math.sqrt(cfg.head_dim)
    out = torch.empty_like(q)
    rmax = torch.empty((slots, n), dtype=torch.float32, device=dev)
    rsum = torch.empty_like(rmax)
    dq, dk, dv = (torch.empty_like(q) for _ in range(3))
    stream = torch.cuda.current_stream(dev).cuda_stream

    def fwd():
        attn_fwd_device(prep, variant, q, k, v, out, rmax, rsum, scale, stream)

    def bwd():
        attn_bwd_device(prep, variant, q, k, v, out, rmax, rsum, g, dq, dk, dv, scale, stream)

    for _ in range(cfg.warmup):
        fwd()
        bwd()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(cfg.runs)]
    for e in ev:
        e[0].record()
        fwd()
        e[1].record()
        bwd()
        e[2].record()
    torch.cuda.synchronize(dev)
    fwd_ms = [a.elapsed_time(b) for a, b, _ in ev]
    bwd_ms = [b.elapsed_time(c) for _, b, c in ev]
    tot_ms = [a.elapsed_time(c) for a, _, c in ev]
    sd = (lambda xs: statistics.stdev(xs) if len(xs) >= 2 else 0.0)
    rec = BenchRecord(variant=variant, mask=label, n=mask.size(), block_i=cfg.block_i, block_j=cfg.block_j,
                      batch=cfg.batch, heads=cfg.heads, runs=cfg.runs, precision=cfg.precision,
                      prepro_ms=prepro_ms, fwd_ms_mean=statistics.fmean(fwd_ms), fwd_ms_std=sd(fwd_ms),
                      bwd_ms_mean=statistics.fmean(bwd_ms), bwd_ms_std=sd(bwd_ms),
                      total_ms_mean=statistics.fmean(tot_ms), counters=prep.counters(variant, slots),
                      block_density=prep.stats.block_density, element_density=prep.stats.element_density)
    if cfg.verify:
        dm = None if variant == Variant.dense else torch.from_numpy(mask.to_dense()).to(dev)
        worst = 0.0
        for s0 in range(slots):
            ref = _torch_reference_forward(q[s0:s0 + 1], k[s0:s0 + 1], v[s0:s0 + 1], scale, dm)
            worst = max(worst, float((out[s0:s0 + 1].float() - ref).abs().max()))
        rec.max_abs_err_vs_oracle = worst
    return rec


def run_bench(cfg: BenchConfig, sink: Optional[Callable[[BenchRecord], None]] = None,
              device: int = 0) -> List[BenchRecord]:
    """run_bench (bench.hpp:472-501) on the B200: one record per (length, variant), plus "+rcm"
    rows when cfg.rcm. Inputs follow make_problem's stream and are rounded to bf16 on upload."""
    import torch

    cfg.validate()
    dev = torch.device("cuda", device)
    free_n = cfg.mask_spec.split("[")[0].split("(")[0] in ("causal", "all-ones", "windowed", "dilated",
                                                             "global", "random")
    lengths = cfg.seq_lengths if free_n else [0]
    records: List[BenchRecord] = []

    def emit(rec):
        if sink:
            sink(rec)
        records.append(rec)

    for length in lengths:
        mask = generate(cfg.mask_spec, length)
        n = mask.size()
        slots = cfg.batch * cfg.heads
        est = estimated_gb(n, cfg.head_dim, slots, cfg.precision)
        if est > cfg.memory_limit_gb:
            raise ValueError(f"estimated working set {est} GiB exceeds limit {cfg.memory_limit_gb} GiB (n={n})")
        if cfg.verify and n > cfg.oracle_limit:
            raise ValueError(f"verification needs n <= {cfg.oracle_limit}, got {n}")
        label = cfg.mask_spec  # MaskSpec::to_string carries no n (generators.hpp:324-362)
        arrs = make_problem(cfg.seed, slots, n, cfg.head_dim)
        tensors = [torch.from_numpy(a).to(dev).to(torch.bfloat16) for a in arrs]
        spec = BlockSpec(cfg.block_i, cfg.block_j)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        prep = preprocess_mask(mask, spec, device=device)
        e1.record()
        torch.cuda.synchronize(dev)
        prepro_ms = e0.elapsed_time(e1)
        for v in cfg.variants:
            emit(_bench_variant(cfg, tensors, mask, prep, prepro_ms, v, label, dev))
        if not cfg.rcm:
            continue
        import time

        t0 = time.perf_counter()
        perm = rcm_order(mask)
        pmask = permute_mask(mask, perm, device=device)
        pprep = preprocess_mask(pmask, spec, device=device)
        rcm_ms = (time.perf_counter() - t0) * 1e3
        # permute_rows (reorder.hpp:167-176) with the device kernel (K5), as bench.hpp:456-458
        ptensors = [permute_rows(t, perm) for t in tensors]
        bw0, bw1 = bandwidth(mask), bandwidth(pmask)
        for v in cfg.variants:
            rec = _bench_variant(cfg, ptensors, pmask, pprep, rcm_ms, v, label + "+rcm", dev)
            rec.bandwidth_before, rec.bandwidth_after = bw0, bw1
            emit(rec)
    return records
