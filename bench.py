"""Benchmark of the B200 masked-attention hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--variant binblk]
    python bench.py --impl reference ...        # the reference's own CPU engine (oracle/_ref)

Default workload: BASELINE config 5 (the metric is quoted "at 1-8 B200", and C5 is the config
sharded over batch x heads): a 1 % structured graph mask (Longformer band w=164 at N=32768,
relabelled by std::shuffle(mt19937_64(3)), then RCM-reordered), B=4 H=32 d=128, binblk.

One step = one blocked_forward over this rank's slots of the config (all B*H slots share one mask
and one MaskPrep, engine.hpp:489-505) with inputs resident in HBM, launched through the C ABI
(bbm_attn_fwd). Under torchrun the config's B*H slots are sharded contiguously over the ranks
([r*S/G, (r+1)*S/G), SURVEY §8e, strong scaling); rank 0 builds the mask metadata once and the
other ranks import it peer to peer (cudaIpc handle + one device-to-device copy over NVLink). No
collective on the data path: the only collectives are the timing barriers, the metadata handle
broadcast before the timed region and the max-over-ranks of the elapsed device time.

Printed on rank 0: ONE JSON line with the contract keys plus roofline / cpu_baseline / e2e /
clocks / dense-run speed-up / preprocessor throughput.

--impl reference never imports paper_2409_15097_b200: it builds the same mask through the
reference's own generators / reorder code (oracle/_ref, compiled from /root/reference headers)
and times the reference's blocked_forward<float> on the host cores.
"""
from __future__ import annotations

import argparse
import importlib.util
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# the pure-Python mt19937_64 (rng.hpp mappings) without importing the package (whose import loads
# libbbm.so, which the reference arm must never touch)
_spec = importlib.util.spec_from_file_location("_bbm_rng", os.path.join(ROOT, "paper_2409_15097_b200", "rng.py"))
_rng = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(_rng)

METRIC = "masked-attn fwd TFLOP/s on executed blocks (ms & speedup vs dense-mask reported beside)"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def alpaca_lengths(total: int, seed: int = 7, lo: int = 64, span: int = 449):
    """Config 2 segment lengths: L_i = 64 + uniform_below(gen, 449) from mt19937_64(seed), the last
    segment truncated so the lengths fill `total`."""
    gen = _rng.MT19937_64(seed)
    out, acc = [], 0
    while acc < total:
        length = min(lo + _rng.uniform_below(gen, span), total - acc)
        out.append(length)
        acc += length
    return out


# BASELINE.json configs: (B, H, d, default variant, description, N)
CONFIGS = {
    "c1": (1, 4, 64, "binblk", "C1 causal B=1 H=4 N=1024 d=64", 1024),
    "c2": (8, 32, 128, "binblk",
           "C2 packed-seq (ALPACA-like lengths U{64..512}, mt19937_64(7)) B=8 H=32 N=4096 d=128", 4096),
    "c3": (1, 32, 128, "binblk", "C3 causal prefix 2048 + MEDUSA[16;15] tree (N=2304) B=1 H=32 d=128", 2304),
    "c4": (1, 16, 64, "dense-binblk", "C4 Longformer window 512 + 128 global, N=16384 B=1 H=16 d=64", 16384),
    "c5": (4, 32, 128, "binblk",
           "C5 1% band (w=164) relabelled by mt19937_64(3), RCM-reordered, N=32768 B=4 H=32 d=128", 32768),
}
VARIANTS = {"dense": 0, "naive": 1, "binblk": 2, "dense-binblk": 3}


def mask_words(name: str, generate, relabel, rcm, permute):
    """The config's mask as reference-layout packed words, composed from four backends so both
    arms build the identical mask: generate(spec, n) -> words, relabel(words, n, seed),
    rcm(words, n) -> forward, permute(words, n, forward). Returns (words, rcm forward or None)."""
    import numpy as np

    n = CONFIGS[name][5]
    if name == "c1":
        return generate("causal", n), None
    if name == "c2":
        return generate("packed-seq[" + ";".join(str(x) for x in alpaca_lengths(n, 7)) + "]", 0), None
    if name == "c3":
        # causal prefix P=2048 + MEDUSA [16;15] tree: prefix rows causal, tree rows see the whole
        # prefix plus their ancestors
        tree = generate("medusa[16;15]", 0)
        t = tree.shape[0]
        wpr = (n + 63) // 64
        dense = np.zeros((n, wpr * 64), bool)
        dense[:2048, :2048] = np.tril(np.ones((2048, 2048), bool))
        dense[2048:, :2048] = True
        tb = np.unpackbits(tree.view(np.uint8), axis=1, bitorder="little")[:, :t].astype(bool)
        dense[2048:, 2048:n] = tb
        return np.packbits(dense, axis=1, bitorder="little").view(np.uint64).reshape(n, wpr), None
    if name == "c4":
        return generate("global(w=512;g=128)", n), None
    if name == "c5":
        shuffled = relabel(generate("windowed(w=164)", n), n, 3)
        fwd = rcm(shuffled, n)
        return permute(shuffled, n, fwd), fwd
    raise SystemExit(f"unknown config {name}")


def bbm_backends(bbm, device: int = 0):
    """mask_words backends on this framework: host generators / relabel / RCM (libbbm host code)
    and the device permute_mask kernel (K6)."""
    def gen(spec, nn):
        return bbm.generate(spec, nn).words

    def relabel(w, nn, seed):
        return bbm.relabel(bbm.Mask(nn, w), seed).words

    def rcm(w, nn):
        return bbm.rcm_order(bbm.Mask(nn, w)).forward

    def permute(w, nn, f):
        return bbm.permute_mask(bbm.Mask(nn, w), bbm.Permutation.from_forward(f), device=device).words

    return gen, relabel, rcm, permute


def make_config(name: str, device: int = 0):
    """(Mask, B, H, d, description) of a config, built with this framework (tests, tools)."""
    import paper_2409_15097_b200 as bbm

    B, H, d, _, desc, n = CONFIGS[name]
    words, _ = mask_words(name, *bbm_backends(bbm, device))
    return bbm.Mask(n, words), B, H, d, desc


def config_dict(name: str, variant: str, world: int, scaling: str) -> dict:
    """The `config` object of the JSON line, identical in both arms."""
    B, H, d, _, desc, n = CONFIGS[name]
    slots = B * H
    return {"workload": desc, "variant": variant, "batch": B, "heads": H, "seq_len": n, "head_dim": d,
            "slots": slots, "tiles": "128x128",
            "parallelism": (f"batch x heads sharded over {world} GPU(s), contiguous slot ranges (strong)"
                            if scaling == "strong" else f"every GPU runs all {slots} slots (weak)"),
            "l2": "inputs > 126 MB L2 (no flush)" if 3 * slots * n * d * 2 > 126e6
            else "inputs < L2: steps back-to-back (L2 warm)"}


def executed_area(cnt, lst, n: int, variant: int) -> float:
    """sum over the kernel's executed 128x128 tiles of rows_in_block * cols_in_block
    (partial tiles count in full); F = 4 * area * d per slot."""
    import numpy as np

    kr = cnt.size
    ext = np.minimum(128, n - np.arange(kr) * 128).astype(np.float64)
    if variant in (0, 1):  # dense / naive: every tile
        return float(ext.sum() ** 2)
    area = 0.0
    for p in range(kr):
        qs = lst[p, : cnt[p]] & 0x7FFFFFFF
        area += ext[p] * float(ext[qs].sum())
    return area


def area_from_words(words, n: int, variant: int) -> float:
    """The same figure from the mask alone (reference arm: the oracle's block sums)."""
    import numpy as np

    import oracle

    sums = oracle.block_sums(words, n, 128, 128)
    ext = np.minimum(128, n - np.arange(sums.shape[0]) * 128).astype(np.float64)
    occ = sums > 0 if variant >= 2 else np.ones_like(sums, bool)
    return float((np.outer(ext, ext) * occ).sum())


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


def cpu_info() -> dict:
    """Host CPU model, physical cores and the threads this process may use."""
    model, cores = None, set()
    try:
        phys = core = None
        with open("/proc/cpuinfo") as f:
            for line in f:
                k, _, v = line.partition(":")
                k, v = k.strip(), v.strip()
                if k == "model name" and model is None:
                    model = v
                elif k == "physical id":
                    phys = v
                elif k == "core id":
                    core = v
                elif not k and phys is not None:
                    cores.add((phys, core))
                    phys = core = None
            if phys is not None:
                cores.add((phys, core))
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = os.cpu_count() or 1
    return {"cpu_model": model, "physical_cores": len(cores) or None, "logical_cpus": os.cpu_count(),
            "usable_threads": usable}


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
                "window": "soak + timed region"}


# ----------------------------------------------------------------------------- reference arm

def ref_mask(name: str):
    """The config's mask built by the reference's own code (oracle/_ref = /root/reference headers
    compiled in place): generators.hpp families, the shuffle relabel through reorder.hpp's
    permute_mask, rcm_order(build_graph) and permute_mask."""
    import oracle

    return mask_words(name, lambda spec, n: oracle.ref_generate(spec, n), oracle.ref_relabel,
                      lambda w, n: oracle.ref_rcm(w, n)[0], oracle.ref_permute_mask)


class RefEngine:
    """The reference's blocked_forward<float> (engine.hpp:282-341) over one slot of make_problem
    inputs, MaskPrep built once (ref_shim.cpp)."""

    def __init__(self, words, n: int, d: int):
        import ctypes as C

        import numpy as np

        import oracle

        self.L = oracle.ref()
        self.words = np.ascontiguousarray(words, dtype=np.uint64)
        q, k, v, _ = oracle.ref_make_problem_f32(1, 1, n, d)
        self.h = self.L.ref_engine_create(self.words.ctypes.data_as(C.POINTER(C.c_uint64)), n, 128, 128,
                                          q.ctypes.data_as(C.POINTER(C.c_float)),
                                          k.ctypes.data_as(C.POINTER(C.c_float)),
                                          v.ctypes.data_as(C.POINTER(C.c_float)), 1, d)
        self.scale = 1.0 / d ** 0.5

    def preprocess_ms(self, reps: int = 1) -> float:
        return self.L.ref_engine_preprocess_ms(self.h, reps)

    def forward(self, variant: int, threads: int) -> float:
        t0 = time.perf_counter()
        self.L.ref_engine_forward(self.h, variant, threads, self.scale)
        return time.perf_counter() - t0

    def close(self):
        if self.h:
            self.L.ref_engine_destroy(self.h)
            self.h = None


def cpu_sample(engine: RefEngine, variant: int, threads: int, budget_s: float, max_slots: int):
    """Time one-slot forwards until `budget_s` (at least one); returns seconds per slot, slots."""
    times = []
    t0 = time.perf_counter()
    while len(times) < max_slots and (not times or time.perf_counter() - t0 < budget_s):
        times.append(engine.forward(variant, threads))
    return statistics.median(times), len(times)


def run_reference_arm(args):
    """--impl reference: the reference CPU implementation on the host cores, rank 0 only. One step
    = blocked_forward<float> over ONE (batch, head) slot of the config (a bounded sample; the
    value is a rate, TFLOP/s on the executed tiles, comparable with the GPU arm's)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    B, H, d, dvar, desc, n = CONFIGS[args.config]
    variant_name = args.variant or dvar
    variant = VARIANTS[variant_name]
    t_setup = time.perf_counter()
    words, _ = ref_mask(args.config)
    flops_slot = 4.0 * area_from_words(words, n, variant) * d
    info = cpu_info()
    threads = info["usable_threads"]
    eng = RefEngine(words, n, d)
    setup_s = time.perf_counter() - t_setup
    try:
        for _ in range(args.warmup):
            eng.forward(variant, threads)
        step_s = [eng.forward(variant, threads) for _ in range(args.steps)]
        pre_ms = eng.preprocess_ms(1)
    finally:
        eng.close()
    ms_step = statistics.mean(step_s) * 1e3
    value = flops_slot / (ms_step * 1e-3) / 1e12
    slots = B * H
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f32 (fp64 accumulate)",
        "data": "synthetic (make_problem uniform[-1,1) inputs, bench.hpp:320-337)",
        "config": config_dict(args.config, variant_name, args.gpus, args.scaling),
        "sample": f"1 of {slots} slots per step (each step = one blocked_forward<float> call; "
                  f"the whole config would take ~{slots * ms_step / 1e3:.1f} s per step)",
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads, "kind": "reference",
                         "sample": f"1 slot per step x {args.steps} steps, blocked_forward<float> "
                                   f"{variant_name} threads={threads}, 128x128 tiles", **info,
                         "preprocess_ms": pre_ms, "setup_s": setup_s},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS))
    ap.add_argument("--variant", default=None, choices=sorted(VARIANTS),
                    help="default: the config's own (dense-binblk for c4, binblk otherwise)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: the config's B*H slots sharded over the ranks (default); "
                         "weak: every rank runs all of them")
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
    ngpu = torch.cuda.device_count()
    oversubscribed = world > ngpu  # test mode: several ranks share a GPU (control collectives on gloo)
    if oversubscribed:
        local = local % max(1, ngpu)
    if world > 1:
        if oversubscribed:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    coll_dev = torch.device("cpu") if oversubscribed else dev  # where the timing reductions run

    B, H, d, dvar, desc, n = CONFIGS[args.config]
    variant_name = args.variant or dvar
    variant = bbm.parse_variant(variant_name)
    scale = 1.0 / d ** 0.5
    slots_total = B * H
    if args.scaling == "strong":
        s0, s1 = bbm.shard_slots(slots_total, world, rank)
    else:
        s0, s1 = 0, slots_total
    slots = s1 - s0
    stream = torch.cuda.current_stream(dev)

    # ---- metadata: rank 0 builds the mask and its prep on its GPU (K1 pack + K2 lists + K3
    # bitmaps from the dense bool mask), the other ranks import it peer to peer
    dense_mask = fwd_perm = None
    t_setup = time.perf_counter()
    if rank == 0:
        words, fwd_perm = mask_words(args.config, *bbm_backends(bbm, local))
        mask = bbm.Mask(n, words)
        dense_mask = torch.from_numpy(mask.to_dense()).to(dev)
        prep = bbm.preprocess_mask(dense_mask, bbm.BlockSpec(128, 128), device=local)
    if world > 1:
        blob = [prep.export_ipc() if rank == 0 else None]
        dist.broadcast_object_list(blob, src=0)
        if rank != 0:
            prep = bbm.import_prep_ipc(blob[0], local)
        dist.barrier()  # every importer has copied the arena before rank 0 may touch its prep
    setup_s = time.perf_counter() - t_setup
    cnt, lst, _ = prep.kernel_lists()
    area = executed_area(cnt, lst, n, int(variant))
    flops = 4.0 * area * d * slots
    # tensor-core work the kernel actually issues: tiles with an empty 64-key half (skipped when at
    # least 10 % of the occupied tiles have one, plan.cu) multiply only the other half
    mma_flops = flops
    if int(variant) in (2, 3):
        hv = prep.tile_halves()
        nhalf = sum(int((hv[p, :c] > 0).sum()) for p, c in enumerate(cnt))
        if nhalf * 10 >= int(cnt.sum()):
            mma_flops = flops - 4.0 * 128 * 64 * d * nhalf * slots  # half of each such tile
    dense_flops = 4.0 * executed_area(cnt, lst, n, 0) * d * slots
    total_flops = 4.0 * area * d * (slots_total if args.scaling == "strong" else slots_total * world)

    # ---- inputs: this rank's slots, uniform[-1,1) bf16, resident in HBM
    g = torch.Generator(device=dev).manual_seed(1234 + s0 + (rank if args.scaling == "weak" else 0))
    q, k, v = ((torch.rand((slots, n, d), generator=g, device=dev) * 2 - 1).to(torch.bfloat16) for _ in range(3))
    out = torch.empty_like(q)
    rmax = torch.empty((slots, n), dtype=torch.float32, device=dev)
    rsum = torch.empty((slots, n), dtype=torch.float32, device=dev)

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
        total_flops *= 2.5

        def step(var=variant):  # noqa: F811
            o_, m_, l_ = fwd_outs[int(var)]
            bbm.attn_bwd_device(prep, var, q, k, v, o_, m_, l_, d_out, *grads, scale, stream.cuda_stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    sampler = ClockSampler(local).start()
    # soak so the sampled clocks reflect the loaded state (short steps alone are sub-ms)
    t_soak = time.perf_counter()
    while time.perf_counter() - t_soak < (0.05 if args.profile else 0.4):
        for _ in range(5):
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
    elapsed_ms = start_all.elapsed_time(end_all)
    launch_ms = [a.elapsed_time(b) for a, b in ev]
    elapsed_ms = max_over_ranks(elapsed_ms, coll_dev)
    ms_step = elapsed_ms / args.steps
    value = total_flops / (ms_step * 1e-3) / 1e12
    if args.profile:
        sampler.stop()
        if rank == 0:
            print(json.dumps({"profile_run": True, "ms_per_step": ms_step, "value": value}))
        if world > 1:
            dist.destroy_process_group()
        return

    extras = {}
    # e2e through the reference-facing host-buffer C ABI, every rank on its own shard, max over
    # ranks (collective timing only)
    if not args.no_e2e and args.which == "fwd":
        extras.update(e2e_all(bbm, prep, variant, q, k, v, slots, n, d, scale, total_flops, args,
                              fwd_perm, coll_dev, world))
    sampler.stop()
    if rank == 0:
        peaks, peak_kind = load_peaks()
        avg_launch = statistics.mean(launch_ms)
        bytes_alg = 4.0 * slots * n * d * 2  # Q, K, V read + O written once (bf16)
        if args.which == "bwd":
            bytes_alg = 8.0 * slots * n * d * 2  # q k v o dO in, dq dk dv out
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
                tr = json.load(f).get(f"{args.config}/{variant_name}/{args.which}")
            if tr and tr.get("slots") == slots:
                traffic = tr.get("dram_bytes_per_launch")
        extras["roofline"] = {
            "bound": bound, "achieved": achieved, "peak": peak, "unit": unit, "frac": achieved / peak,
            "traffic": traffic, "peak_source": f"{peak_kind} (MEASURED_PEAKS.json burst)",
            "kernel": "attn_fwd_kernel" if args.which == "fwd" else "attn_bwd_kernel (dq + dkdv)",
            "algorithmic_bytes_per_launch": bytes_alg, "flops_per_launch": flops,
            "mma_flops_per_launch": mma_flops,
            "flops_note": "flops_per_launch counts every executed 128x128 tile in full (SURVEY 8d); "
                          "mma_flops_per_launch is the tensor work issued (64-key halves no row sees are "
                          "skipped)",
            "tensor_frac": (flops / (avg_launch * 1e-3) / 1e12) / peaks["bf16_tflops"],
            "hbm_frac": (bytes_alg / (avg_launch * 1e-3) / 1e9) / peaks["hbm_gbs"],
            "avg_launch_ms": avg_launch, "slots_per_launch": slots,
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
                                    "speedup_vs_dense": dense_ms / (avg_launch if world > 1 else ms_step),
                                    "ideal_speedup_by_tiles": dense_flops / flops}
        if args.which == "fwd":
            extras["preprocess"] = preprocess_measure(bbm, prep, dense_mask, stream, n, step, ms_step)
        if args.which == "fwd" and fwd_perm is not None:
            # f2: the same forward on ORIGINAL-order inputs with the RCM permutation applied on the
            # device (bbm_attn_fwd_gather_ex): permute passes around the plain kernel (mode 1), the
            # in-kernel TMA tile::gather4 (mode 2), the hybrid (mode 3: K/V passes, Q/O in the
            # kernel) and the default in-kernel LSU gather (mode 4), against the pre-permuted
            # forward above
            rows = torch.from_numpy(np.ascontiguousarray(fwd_perm, dtype=np.int32)).to(dev)
            og = torch.empty_like(q)
            rcm = {}
            for mode, key in ((1, "passes"), (2, "in_kernel_tma"), (3, "hybrid"), (4, "in_kernel_lsu")):
                def gstep(mode=mode):
                    bbm.attn_fwd_device(prep, variant, q, k, v, og, rmax, rsum, scale, stream.cuda_stream,
                                        rows=rows, gather_mode=mode)

                for _ in range(3):
                    gstep()
                rcm[key] = device_ms(stream, gstep, max(5, args.steps))
            p_ms = device_ms(stream, step, max(5, args.steps))
            extras["fwd_device_rcm"] = {
                "ms_per_step": rcm["in_kernel_lsu"], "pre_permuted_ms_per_step": p_ms,
                "ratio_vs_pre_permuted": rcm["in_kernel_lsu"] / p_ms,
                "tflops": flops / (rcm["in_kernel_lsu"] * 1e-3) / 1e12,
                "hybrid_ms_per_step": rcm["hybrid"], "passes_ms_per_step": rcm["passes"],
                "in_kernel_tma_ms_per_step": rcm["in_kernel_tma"],
                "note": "original-order Q/K/V resident in HBM; default path (bbm_attn_fwd_gather, mode 4): every "
                        "Q/K/V row gathered inside the kernel by LSU cp.async (two producer warps), O rows "
                        "written to their tokens by the epilogue threads, no scratch; hybrid (mode 3): K/V "
                        "permuted by passes, Q gathered / O scattered with TMA tile::gather4 / scatter4; passes "
                        "(mode 1): Q/K/V permuted, plain kernel, O and row stats scattered back; in_kernel_tma "
                        "(mode 2): every row gathered with tile::gather4 (bound by the TMA instruction rate)"}
            del og
        if not args.no_cpu_baseline and world == 1 and args.which == "fwd":
            try:
                info = cpu_info()
                threads = info["usable_threads"]
                eng = RefEngine(mask.words, n, d)
                try:
                    eng.forward(int(variant), threads)  # warm
                    sec_slot, done = cpu_sample(eng, int(variant), threads, 15.0, slots)
                    ref_pre_ms = eng.preprocess_ms(1)
                finally:
                    eng.close()
                extras["cpu_baseline"] = {
                    "value": (flops / slots) / sec_slot / 1e12, "unit": "TFLOP/s", "cores": threads,
                    "kind": "reference",
                    "sample": f"{done} one-slot blocked_forward<float> calls (~15 s), {variant_name}, "
                              f"threads={threads}, 128x128 tiles; whole config ~{sec_slot * slots:.1f} s",
                    **info, "preprocess_ms_reference": ref_pre_ms,
                }
            except Exception as e:  # noqa: BLE001
                extras["cpu_baseline"] = {"value": None, "unavailable": str(e)}
        extras["clocks"] = sampler.summary(t_soak, t1)
        extras["setup_s"] = setup_s

    if rank == 0:
        line = {
            "metric": METRIC if args.which == "fwd" else METRIC.replace("fwd", "bwd (5-GEMM FLOPs)"),
            "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (uniform[-1,1) bf16 inputs)",
            "config": config_dict(args.config, variant_name, world, args.scaling),
            "gpu_launches": args.steps * (1 if args.which == "fwd" else 3),
        }
        if oversubscribed:
            line["note"] = f"TEST MODE: {world} ranks on {ngpu} GPU(s) (gloo control collectives); not a scaling number"
        line.update(extras)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def device_ms(stream, fn, reps: int) -> float:
    """Device time of `reps` back-to-back calls of fn: the stream is first given ~20 ms of sleep so
    the host enqueues every call before the device reaches them (host-side call overhead, which
    exceeds a small kernel, then cannot starve the device between the events)."""
    import torch

    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    torch.cuda._sleep(int(20e-3 * 1.9e9))
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def preprocess_measure(bbm, prep, dense_mask, stream, n, step, fwd_ms):
    """The per-batch path: bbm_prep_update_bool_device rebuilds the prep from a dense bool mask on
    the device (one fused launch: pack + sums + lists + bitmaps + order, no host round trip);
    then the same with a forward after every update, alternating two different masks (the
    forward re-plans on the device for each new mask version)."""
    reps = 20
    for _ in range(3):
        prep.update(dense_mask, stream.cuda_stream)
    pre_ms = device_ms(stream, lambda: prep.update(dense_mask, stream.cuda_stream), reps)
    # a second mask of the same size: the first one's transpose (same density, other lists)
    other = dense_mask.t().contiguous()
    masks = [other, dense_mask]
    state = {"i": 0}

    def both():
        prep.update(masks[state["i"] % 2], stream.cuda_stream)
        step()
        state["i"] += 1

    both()
    both_ms = device_ms(stream, both, reps)
    if state["i"] % 2 == 1:  # leave the prep on the config's own mask
        prep.update(dense_mask, stream.cuda_stream)
    del other
    return {"ms": pre_ms, "input": f"dense bool mask {n}x{n} on device",
            "gbs_bool_read": n * n / (pre_ms * 1e-3) / 1e9,
            "hbm_frac_bool_read": n * n / (pre_ms * 1e-3) / 1e9 / load_peaks()[0]["hbm_gbs"],
            "kernels": "prep_fused_kernel (one launch)",
            "update_plus_forward_ms": both_ms, "forward_ms": fwd_ms,
            "update_plus_forward_note": "fresh mask every step (alternating the mask and its transpose); "
                                        "the forward's launch plan is rebuilt on the device each time; "
                                        "device time (host enqueue hidden behind a sleep)"}


def e2e_all(bbm, prep, variant, q, k, v, slots, n, d, scale, total_flops, args, fwd_perm, dev, world):
    """e2e through the reference-facing host-buffer C ABI: Q/K/V from pinned host memory, H2D,
    the kernel and D2H of O and the row statistics inside the timed call, every step.

    e2e      bbm_run_attention_host_f32: the reference's own types (run_attention<float>,
             engine.hpp:489-505): per-slot Matrix<float> buffers in, float out, double row stats
    e2e_bf16 bbm_attn_fwd_host_bf16: bf16 host buffers (half the PCIe bytes)
    e2e_rcm  (C5) the reordered pipeline from ORIGINAL-order bf16 buffers (device gather/scatter)
    Times are max over ranks."""
    import ctypes as C

    import numpy as np
    import torch

    from paper_2409_15097_b200 import _lib

    reps = max(3, min(args.steps, 5))
    res = {}

    def timed(call):
        call()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        for _ in range(reps):
            call()
        ms = (time.perf_counter() - t0) / reps * 1e3
        return max_over_ranks(ms, dev)

    # f32 per-slot (the reference signature)
    hq, hk, hv = (t.float().cpu().pin_memory() for t in (q, k, v))
    ho = torch.empty((slots, n, d), dtype=torch.float32).pin_memory()
    hm = torch.empty((slots, n), dtype=torch.float64).pin_memory()
    hs = torch.empty((slots, n), dtype=torch.float64).pin_memory()
    arr = lambda t, per: (C.c_void_p * slots)(*[t.data_ptr() + i * per for i in range(slots)])  # noqa: E731
    pq, pk, pv, po = (arr(t, n * d * 4) for t in (hq, hk, hv, ho))
    pm, ps = arr(hm, n * 8), arr(hs, n * 8)

    def call_f32():
        _lib.check(_lib.lib.bbm_run_attention_host_f32(prep.handle.h, int(variant), pq, pk, pv, po, pm, ps,
                                                       slots, d, scale))

    ms = timed(call_f32)
    res["e2e"] = {"value": total_flops / (ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": ms,
                  "h2d_bytes_per_step": 3 * slots * n * d * 4,
                  "d2h_bytes_per_step": slots * n * d * 4 + 2 * slots * n * 8,
                  "path": "bbm_run_attention_host_f32 (C ABI of run_attention<float>: per-slot float host "
                          "buffers, pinned; ~70% of each chunk's slots rounded to bf16 by host threads into "
                          "pinned staging, the rest converted on the device, finiteness checked on both; "
                          "float out, double row stats; synchronous)"}
    del hq, hk, hv, ho, hm, hs

    u16 = C.POINTER(C.c_uint16)
    f32 = C.POINTER(C.c_float)
    bq, bk, bv = (t.cpu().pin_memory() for t in (q, k, v))
    bo = torch.empty_like(bq).pin_memory()
    bm = torch.empty((slots, n), dtype=torch.float32).pin_memory()
    bs = torch.empty((slots, n), dtype=torch.float32).pin_memory()
    ptrs = [C.cast(t.data_ptr(), u16) for t in (bq, bk, bv, bo)] + [C.cast(t.data_ptr(), f32) for t in (bm, bs)]

    def call_bf16():
        _lib.check(_lib.lib.bbm_attn_fwd_host_bf16(prep.handle.h, int(variant), *ptrs, slots, d, scale))

    ms = timed(call_bf16)
    h2d, d2h = 3 * slots * n * d * 2, slots * n * d * 2 + 2 * slots * n * 4
    res["e2e_bf16"] = {"value": total_flops / (ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": ms,
                       "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                       "path": "bbm_attn_fwd_host_bf16 (pinned bf16 host buffers, synchronous)"}
    if fwd_perm is not None and world == 1:
        fwd = np.ascontiguousarray(fwd_perm, dtype=np.uint32)

        def call_rcm():
            _lib.check(_lib.lib.bbm_attn_fwd_rcm_host_bf16(prep.handle.h, int(variant),
                                                           fwd.ctypes.data_as(C.POINTER(C.c_uint32)), *ptrs,
                                                           slots, d, scale))

        ms = timed(call_rcm)
        res["e2e_rcm"] = {"value": total_flops / (ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": ms,
                          "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                          "path": "bbm_attn_fwd_rcm_host_bf16 (original token order; RCM gather/scatter "
                                  "on the device)"}
    return res


if __name__ == "__main__":
    main()
