"""Benchmark of the B200 masked-attention hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--variant binblk]
    python bench.py --impl reference ...        # the reference's own CPU engine (oracle/_ref)

One step = one blocked_forward over the whole config (all B*H slots share one mask and one
MaskPrep, engine.hpp:489-505) with inputs resident in HBM, launched through the C ABI
(bbm_attn_fwd). Under torchrun each rank runs its own full config on its own GPU (weak scaling,
disjoint slot ranges of a virtual global batch; no collective on the data path — the only
collectives are the timing barrier and the max-over-ranks of the elapsed time).

Printed on rank 0: ONE JSON line with the contract keys plus roofline / cpu_baseline / e2e /
clocks / dense-run speedup / preprocessor throughput.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2409_15097_b200.rng import MT19937_64, uniform_below  # noqa: E402

METRIC = "masked-attn fwd TFLOP/s on executed blocks (ms & speedup vs dense-mask reported beside)"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def alpaca_lengths(total: int, seed: int = 7, lo: int = 64, span: int = 449):
    """Config 2 segment lengths: L_i = 64 + uniform_below(gen, 449) from mt19937_64(seed), the last
    segment truncated so the lengths fill `total`."""
    gen = MT19937_64(seed)
    out, acc = [], 0
    while acc < total:
        length = min(lo + uniform_below(gen, span), total - acc)
        out.append(length)
        acc += length
    return out


RCM_PERM = {}  # config -> RCM permutation (new -> old) of its reordered mask


def make_config(name: str):
    """BASELINE.json configs -> (mask, B, H, d, description). C2 is the headline workload."""
    import paper_2409_15097_b200 as bbm

    if name == "c1":
        return bbm.gen_causal(1024), 1, 4, 64, "C1 causal B=1 H=4 N=1024 d=64"
    if name == "c2":
        return (bbm.gen_packed_sequential(alpaca_lengths(4096, 7)), 8, 32, 128,
                "C2 packed-seq (ALPACA-like lengths U{64..512}, mt19937_64(7)) B=8 H=32 N=4096 d=128")
    if name == "c3":
        # causal prefix P=2048 + MEDUSA [16;15] tree: prefix rows causal, tree rows see the whole
        # prefix plus their ancestors
        tree = bbm.gen_medusa([16, 15])
        t = tree.size()
        n = 2048 + t
        m = bbm.Mask(n)
        dense = m.to_dense()
        import numpy as np

        dense[:2048, :2048] = np.tril(np.ones((2048, 2048), bool))
        dense[2048:, :2048] = True
        dense[2048:, 2048:] = tree.to_dense()
        return (bbm.Mask.from_dense(dense), 1, 32, 128,
                f"C3 causal prefix 2048 + MEDUSA[16;15] tree (N={n}) B=1 H=32 d=128")
    if name == "c4":
        return (bbm.gen_longformer_global(16384, 512, 128), 1, 16, 64,
                "C4 Longformer window 512 + 128 global, N=16384 H=16 d=64")
    if name == "c5":
        base = bbm.gen_longformer_windowed(32768, 164)
        shuffled = bbm.relabel(base, 3)
        perm = bbm.rcm_order(shuffled)
        RCM_PERM["c5"] = perm
        return (bbm.permute_mask(shuffled, perm), 4, 32, 128,
                "C5 1% band (w=164) relabelled by mt19937_64(3), RCM-reordered, N=32768 B=4 H=32 d=128")
    raise SystemExit(f"unknown config {name}")


def executed_flops(prep, slots: int, d: int, variant: int) -> float:
    """F = slots * sum over executed tiles of 4 * rows_in_block * cols_in_block * d,
    at the kernel's 128x128 tiling (partial tiles count in full)."""
    import numpy as np

    n = prep.n_tokens
    cnt, lst, _ = prep.kernel_lists()
    kr = cnt.size
    ext = np.minimum(128, n - np.arange(kr) * 128).astype(np.float64)
    if variant in (0, 1):  # dense / naive: every tile
        area = float(ext.sum() ** 2)
    else:
        area = 0.0
        for p in range(kr):
            qs = lst[p, : cnt[p]] & 0x7FFFFFFF
            area += ext[p] * float(ext[qs].sum())
    return 4.0 * area * d * slots


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank float over the default process group (the contract's max-over-ranks
    device time); identity when torch.distributed is not initialised."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f), "measured"
    return PEAKS_FALLBACK, "fallback"


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons while the GPU is under load."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples = []
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:  # noqa: BLE001
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                sm = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                rs = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((time.perf_counter(), sm, rs))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.005)

    def start(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def stop(self):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self, t0: float, t1: float):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"], "samples": 0}
        inside = [s for s in self.samples if t0 <= s[0] <= t1] or self.samples
        mhz = statistics.median(s[1] for s in inside)
        bits = 0
        for s in inside:
            bits |= s[2]
        reasons = sorted({name for b, name in self.REASONS.items() if bits & b and name != "gpu_idle"})
        return {"sm_mhz": mhz, "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(inside),
                "window": "soak + timed region (timed steps are sub-ms)"}


def cpu_reference_run(mask, slots_total, d, variant, budget_s, threads, min_slots=1):
    """The reference's own CPU engine (blocked_forward<float>, engine.hpp:282-341, compiled from
    the reference headers into oracle/_ref) over a bounded sample of the workload's slots.
    Returns (seconds per slot, slots timed, preprocess ms)."""
    import numpy as np

    import oracle

    if not oracle.ref_available():
        raise RuntimeError("oracle/_ref/libbbm_ref.so not built")
    L = oracle.ref()
    n = mask.size()
    # one slot of make_problem-style inputs (values do not change the work: counters and tile
    # walk depend on the mask only, engine.hpp:47-48)
    q, k, v, _ = oracle.ref_make_problem_f32(1, 1, n, d)
    words = np.ascontiguousarray(mask.words)
    import ctypes as C

    h = L.ref_engine_create(words.ctypes.data_as(C.POINTER(C.c_uint64)), n, 128, 128,
                            q.ctypes.data_as(C.POINTER(C.c_float)), k.ctypes.data_as(C.POINTER(C.c_float)),
                            v.ctypes.data_as(C.POINTER(C.c_float)), 1, d)
    try:
        prepro_ms = L.ref_engine_preprocess_ms(h, 1)
        L.ref_engine_forward(h, variant, threads, 1.0 / d ** 0.5)  # warm
        t0 = time.perf_counter()
        done = 0
        while done < slots_total and (done < min_slots or time.perf_counter() - t0 < budget_s):
            L.ref_engine_forward(h, variant, threads, 1.0 / d ** 0.5)
            done += 1
        el = time.perf_counter() - t0
    finally:
        L.ref_engine_destroy(h)
    return el / done, done, prepro_ms


def run_reference_arm(args):
    """--impl reference: the reference CPU implementation on the host cores, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    mask, B, H, d, desc = make_config(args.config)
    slots = B * H
    variant = {"dense": 0, "naive": 1, "binblk": 2, "dense-binblk": 3}[args.variant]
    import numpy as np  # noqa: F401

    import paper_2409_15097_b200 as bbm

    # executed-tile FLOPs from the mask alone (host oracle-free computation of the same figure)
    sums = __import__("oracle").block_sums(mask.words, mask.size(), 128, 128)
    n = mask.size()
    ext = np.minimum(128, n - np.arange(sums.shape[0]) * 128).astype(np.float64)
    occ = sums > 0 if variant >= 2 else np.ones_like(sums, bool)
    flops_slot = 4.0 * float((np.outer(ext, ext) * occ).sum()) * d
    threads = os.cpu_count() or 1
    per_step_budget = max(2.0, 60.0 / max(1, args.steps + args.warmup))
    for _ in range(args.warmup):
        cpu_reference_run(mask, 1, d, variant, 0.0, threads)
    times = []
    sample_slots = []
    for _ in range(args.steps):
        sec_per_slot, done, _ = cpu_reference_run(mask, slots, d, variant, per_step_budget, threads)
        times.append(sec_per_slot)
        sample_slots.append(done)
    sec_slot = statistics.median(times)
    value = flops_slot / sec_slot / 1e12
    ms_step = sec_slot * slots * 1e3
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32 (fp64 accumulate)", "data": "synthetic",
        "config": {"workload": desc, "variant": args.variant, "slots": slots, "tiles": "128x128",
                   "extrapolated_from_slots_per_step": sample_slots},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads, "kind": "reference",
                         "sample": f"{min(sample_slots)}-{max(sample_slots)} of {slots} slots per step, "
                                   f"blocked_forward<float> threads={threads}, ms_per_step extrapolated x{slots}"},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    del bbm


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--variant", default="binblk", choices=["dense", "naive", "binblk", "dense-binblk"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile", action="store_true", help="minimal run for ncu (no extras)")
    ap.add_argument("--pass", dest="which", default="fwd", choices=["fwd", "bwd"],
                    help="fwd: the BASELINE metric; bwd: blocked_backward over the same tiles")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    if args.impl == "reference":
        run_reference_arm(args)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2409_15097_b200 as bbm

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    mask, B, H, d, desc = make_config(args.config)
    slots = B * H
    n = mask.size()
    variant = bbm.parse_variant(args.variant)
    scale = 1.0 / d ** 0.5

    # metadata: built once per GPU from the dense bool mask on the device (K1+K2+lists+bitmaps),
    # exactly as shared by every slot (engine.hpp:68-70)
    dense_mask = torch.from_numpy(mask.to_dense()).to(dev)
    prep = bbm.preprocess_mask(dense_mask, bbm.BlockSpec(128, 128), device=local)
    flops = executed_flops(prep, slots, d, int(variant))
    dense_flops = executed_flops(prep, slots, d, 0)

    # inputs: this rank's slots of the virtual global batch, uniform[-1,1) bf16, resident in HBM
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    q, k, v = ((torch.rand((slots, n, d), generator=g, device=dev) * 2 - 1).to(torch.bfloat16) for _ in range(3))
    out = torch.empty_like(q)
    rmax = torch.empty((slots, n), dtype=torch.float32, device=dev)
    rsum = torch.empty((slots, n), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step(var=variant):
        bbm.attn_fwd_device(prep, var, q, k, v, out, rmax, rsum, scale, stream.cuda_stream)

    if args.which == "bwd":
        # blocked_backward (engine.hpp:346-471) from this forward's output and row statistics;
        # FLOPs counted the standard way (5 GEMMs per executed tile = 2.5x the forward's),
        # although the two deterministic kernels recompute S and dP (7 GEMMs)
        d_out = (torch.rand((slots, n, d), generator=g, device=dev) * 2 - 1).to(torch.bfloat16)
        grads = [torch.empty_like(q) for _ in range(3)]
        fwd_outs = {}
        for var in {int(variant), 0}:
            o_, m_, l_ = torch.empty_like(q), torch.empty_like(rmax), torch.empty_like(rsum)
            bbm.attn_fwd_device(prep, var, q, k, v, o_, m_, l_, scale, stream.cuda_stream)
            fwd_outs[var] = (o_, m_, l_)
        flops *= 2.5
        dense_flops *= 2.5

        def step(var=variant):  # noqa: F811
            o_, m_, l_ = fwd_outs[int(var)]
            bbm.attn_bwd_device(prep, var, q, k, v, o_, m_, l_, d_out, *grads, scale, stream.cuda_stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    sampler = ClockSampler(local).start()
    # soak so the sampled clocks reflect the loaded state (timed steps alone are sub-ms)
    t_soak = time.perf_counter()
    while time.perf_counter() - t_soak < (0.05 if args.profile else 0.4):
        for _ in range(20):
            step()
        torch.cuda.synchronize()

    # ---- timed region: K steps, barrier + synchronize on both sides, per-launch CUDA events
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    start_all = torch.cuda.Event(enable_timing=True)
    end_all = torch.cuda.Event(enable_timing=True)
    start_all.record(stream)
    for i in range(args.steps):
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    end_all.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t1 = time.perf_counter()
    sampler.stop()
    elapsed_ms = start_all.elapsed_time(end_all)
    launch_ms = [a.elapsed_time(b) for a, b in ev]
    elapsed_ms = max_over_ranks(elapsed_ms, dev)
    ms_step = elapsed_ms / args.steps
    value = world * flops / (ms_step * 1e-3) / 1e12
    if args.profile:
        if rank == 0:
            print(json.dumps({"profile_run": True, "ms_per_step": ms_step, "value": value}))
        if world > 1:
            dist.destroy_process_group()
        return

    extras = {}
    if rank == 0:
        peaks, peak_kind = load_peaks()
        avg_launch = statistics.mean(launch_ms)
        bytes_alg = 4.0 * slots * n * d * 2  # Q, K, V read + O written once (bf16)
        t_tensor = flops / (peaks["bf16_tflops"] * 1e12)
        t_hbm = bytes_alg / (peaks["hbm_gbs"] * 1e9)
        if t_hbm > t_tensor:
            bound, achieved, peak, unit = "hbm", bytes_alg / (avg_launch * 1e-3) / 1e9, peaks["hbm_gbs"], "GB/s"
        else:
            bound, achieved, peak, unit = "tensor", flops / (avg_launch * 1e-3) / 1e12, peaks["bf16_tflops"], "TFLOP/s"
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tpath):
            with open(tpath) as f:
                tr = json.load(f).get(f"{args.config}/{args.variant}")
            if tr:
                traffic = tr.get("dram_bytes_per_launch")
        extras["roofline"] = {
            "bound": bound, "achieved": achieved, "peak": peak, "unit": unit, "frac": achieved / peak,
            "traffic": traffic, "peak_source": f"{peak_kind} (MEASURED_PEAKS.json burst)",
            "algorithmic_bytes_per_launch": bytes_alg, "flops_per_launch": flops,
            "tensor_frac": (flops / (avg_launch * 1e-3) / 1e12) / peaks["bf16_tflops"],
            "hbm_frac": (bytes_alg / (avg_launch * 1e-3) / 1e9) / peaks["hbm_gbs"],
            "avg_launch_ms": avg_launch,
        }
        # dense-mask run of the same kernel (all tiles, no mask reads)
        for _ in range(2):
            step(bbm.Variant.dense)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        e0.record(stream)
        for _ in range(reps):
            step(bbm.Variant.dense)
        e1.record(stream)
        torch.cuda.synchronize()
        dense_ms = e0.elapsed_time(e1) / reps
        extras["dense_mask_run"] = {"ms_per_step": dense_ms, "tflops": dense_flops / (dense_ms * 1e-3) / 1e12,
                                    "speedup_vs_dense": dense_ms / ms_step,
                                    "ideal_speedup_by_tiles": dense_flops / flops}
        # preprocessor: per-batch rebuild of the kernel metadata from the dense bool mask
        if args.which == "bwd":
            args.no_e2e = args.no_cpu_baseline = True
        for _ in range(3):
            prep_update(prep, dense_mask, stream)
        torch.cuda.synchronize()
        e0.record(stream)
        reps = 20
        for _ in range(reps):
            prep_update(prep, dense_mask, stream)
        e1.record(stream)
        torch.cuda.synchronize()
        pre_ms = e0.elapsed_time(e1) / reps
        extras["preprocess"] = {"ms": pre_ms, "input": f"dense bool mask {n}x{n} on device",
                                "gbs_bool_read": n * n / (pre_ms * 1e-3) / 1e9,
                                "kernels": "pack_bool_sums128 + rowmeta + compact_bitmaps + finalize"}
        # e2e: the same forward through the host-buffer C ABI call, H2D + D2H inside the region
        if not args.no_e2e:
            extras["e2e"] = e2e_measure(prep, variant, q, k, v, slots, n, d, scale, flops, args.steps)
            if args.config in RCM_PERM:  # the whole reordered pipeline from original-order buffers
                extras["e2e_rcm"] = e2e_measure(prep, variant, q, k, v, slots, n, d, scale, flops, args.steps,
                                                forward=RCM_PERM[args.config].forward)
        if not args.no_cpu_baseline and world == 1:
            try:
                threads = os.cpu_count() or 1
                sec_slot, done, ref_pre_ms = cpu_reference_run(mask, slots, d, int(variant), 15.0, threads)
                cpu_val = (flops / slots) / sec_slot / 1e12
                extras["cpu_baseline"] = {
                    "value": cpu_val, "unit": "TFLOP/s", "cores": threads, "kind": "reference",
                    "sample": f"{done} of {slots} slots (one slot's inputs re-run), reference "
                              f"blocked_forward<float> {args.variant} threads={threads}, 128x128 tiles",
                    "ms_per_step_extrapolated": sec_slot * slots * 1e3,
                    "preprocess_ms_reference": ref_pre_ms,
                }
            except Exception as e:  # noqa: BLE001
                extras["cpu_baseline"] = {"value": None, "unavailable": str(e)}
        extras["clocks"] = sampler.summary(t_soak, t1)

    if rank == 0:
        line = {
            "metric": METRIC if args.which == "fwd" else METRIC.replace("fwd", "bwd (5-GEMM FLOPs)"),
            "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (uniform[-1,1) bf16 inputs)",
            "config": {"workload": desc, "variant": args.variant, "batch": B, "heads": H, "seq_len": n,
                       "head_dim": d, "slots_per_gpu": slots, "global_slots": slots * world,
                       "tiles": "128x128", "parallelism": f"slot shards x{world} (weak)",
                       "l2": "inputs > 126 MB L2 (no flush)" if 3 * slots * n * d * 2 > 126e6
                       else "inputs < L2: steps back-to-back (L2 warm)"},
            "gpu_launches": args.steps,
        }
        line.update(extras)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def prep_update(prep, dense_mask, stream):
    import ctypes as C

    from paper_2409_15097_b200 import _lib

    _lib.check(_lib.lib.bbm_prep_update_bool_device(prep.handle.h, C.c_void_p(dense_mask.data_ptr()),
                                                     dense_mask.stride(0), C.c_void_p(stream.cuda_stream)))


def e2e_measure(prep, variant, q, k, v, slots, n, d, scale, flops, steps, forward=None):
    """bbm_attn_fwd_host_bf16 with pinned host buffers: H2D of Q/K/V, the kernel, D2H of O and the
    row statistics, all inside the timed call. With `forward` (an RCM permutation), the
    reordered pipeline bbm_attn_fwd_rcm_host_bf16 instead: original-order buffers, the device
    gathers / scatters rows around the kernel."""
    import ctypes as C

    import torch

    from paper_2409_15097_b200 import _lib

    hq, hk, hv = (t.cpu().pin_memory() for t in (q, k, v))
    ho = torch.empty_like(hq).pin_memory()
    hmax = torch.empty((slots, n), dtype=torch.float32).pin_memory()
    hsum = torch.empty((slots, n), dtype=torch.float32).pin_memory()

    import numpy as np

    fwd = None if forward is None else np.ascontiguousarray(forward, dtype=np.uint32)

    def call():
        u16 = C.POINTER(C.c_uint16)
        f32 = C.POINTER(C.c_float)
        if fwd is not None:
            _lib.check(_lib.lib.bbm_attn_fwd_rcm_host_bf16(
                prep.handle.h, int(variant), fwd.ctypes.data_as(C.POINTER(C.c_uint32)),
                C.cast(hq.data_ptr(), u16), C.cast(hk.data_ptr(), u16), C.cast(hv.data_ptr(), u16),
                C.cast(ho.data_ptr(), u16), C.cast(hmax.data_ptr(), f32), C.cast(hsum.data_ptr(), f32),
                slots, d, scale))
            return
        _lib.check(_lib.lib.bbm_attn_fwd_host_bf16(
            prep.handle.h, int(variant), C.cast(hq.data_ptr(), u16), C.cast(hk.data_ptr(), u16),
            C.cast(hv.data_ptr(), u16), C.cast(ho.data_ptr(), u16), C.cast(hmax.data_ptr(), f32),
            C.cast(hsum.data_ptr(), f32), slots, d, scale))

    call()
    reps = max(3, min(steps, 10))
    t0 = time.perf_counter()
    for _ in range(reps):
        call()
    ms = (time.perf_counter() - t0) / reps * 1e3
    h2d = 3 * slots * n * d * 2
    d2h = slots * n * d * 2 + 2 * slots * n * 4
    return {"value": flops / (ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": ms,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "path": ("bbm_attn_fwd_rcm_host_bf16 (original token order; device gather/scatter)" if fwd is not None
                     else "bbm_attn_fwd_host_bf16") + " (C ABI, pinned host buffers, synchronous)"}


if __name__ == "__main__":
    main()
