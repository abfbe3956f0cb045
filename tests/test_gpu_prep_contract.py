"""The reference's MaskPrep contract on the B200 (-m gpu): "built once and shared across heads,
runs and both passes" (engine.hpp:68-70), "safe to call from any number of threads concurrently;
no shared mutable state".

* an update (bbm_prep_update_*) behaves exactly like a fresh preprocess of the new mask: device
  launches, getters, counters and the multi-GPU driver's replicas all follow it;
* one prep used from two streams at once gives bitwise the single-stream results;
* the prep's metadata moves between processes (cudaIpc export / import) bit for bit;
* the reference-signature host path (per-slot Matrix<float>, bbm_run_attention_host_f32) equals
  the device path, and host paths reject non-finite inputs like require_finite.
"""
import ctypes as C
import multiprocessing as mp
import os

import numpy as np
import pytest

import oracle
import paper_2409_15097_b200 as bbm
from paper_2409_15097_b200 import _lib

pytestmark = pytest.mark.gpu


def dev_inputs(cuda, slots, n, d, seed=1):
    import torch

    g = torch.Generator(device=cuda).manual_seed(seed)
    return [(torch.rand((slots, n, d), generator=g, device=cuda) * 2 - 1).to(torch.bfloat16) for _ in range(3)]


def fwd(prep, variant, q, k, v, stream=None, scale=None):
    import torch

    out = torch.empty_like(q)
    m = torch.empty(q.shape[:2], dtype=torch.float32, device=q.device)
    l = torch.empty_like(m)
    bbm.attn_fwd_device(prep, variant, q, k, v, out, m, l,
                        1 / np.sqrt(q.shape[-1]) if scale is None else scale, stream)
    return out, m, l


def bits(t):
    import torch

    return t.contiguous().view(torch.int32 if t.element_size() == 4 else torch.int16)


def same(a, b):
    """Bitwise equality of tuples of tensors (NaN-safe, -0 != +0)."""
    import torch

    return all(torch.equal(bits(x), bits(y)) for x, y in zip(a, b))


def masks_pair(n):
    a = bbm.gen_packed_sequential([n // 4, n // 2, n - n // 4 - n // 2])
    b = bbm.gen_longformer_global(n, 97, 33)
    return a, b


@pytest.mark.parametrize("variant", [bbm.Variant.binblk, bbm.Variant.dense_binblk, bbm.Variant.naive_masked])
def test_update_equals_fresh_prep(cuda, variant):
    import torch

    n, d, slots = 1000, 128, 3
    a, b = masks_pair(n)
    q, k, v = dev_inputs(cuda, slots, n, d)
    prep = bbm.preprocess_mask(a, bbm.BlockSpec(128, 128))
    first = fwd(prep, variant, q, k, v)
    fresh_b = bbm.preprocess_mask(b, bbm.BlockSpec(128, 128))
    want_b = fwd(fresh_b, variant, q, k, v)
    # update to b on the device (dense bool), forward again with the SAME prep: no host sync between
    prep.update(torch.from_numpy(b.to_dense()).to(cuda))
    got_b = fwd(prep, variant, q, k, v)
    torch.cuda.synchronize()
    assert same(got_b, want_b)
    assert not same(got_b, first)
    # and back (packed words path)
    prep.update(torch.from_numpy(a.words.view(np.int64)).to(cuda))
    assert same(fwd(prep, variant, q, k, v), first)


def test_update_refreshes_getters_and_counters(cuda):
    import torch

    n = 777
    a, b = masks_pair(n)
    for spec in (bbm.BlockSpec(128, 128), bbm.BlockSpec(64, 32)):
        prep = bbm.preprocess_mask(a, spec)
        prep.update(torch.from_numpy(b.to_dense()).to(cuda))
        assert np.array_equal(prep.sums.values, oracle.block_sums(b.words, n, spec.block_i, spec.block_j))
        fresh = bbm.preprocess_mask(b, spec)
        assert prep.occupancy == fresh.occupancy
        assert prep.runs == fresh.runs
        assert prep.stats == fresh.stats
        for var in bbm.Variant:
            assert prep.counters(var, 5) == fresh.counters(var, 5)
        cnt, lst, order = prep.kernel_lists()
        c2, l2, o2 = fresh.kernel_lists()
        assert np.array_equal(cnt, c2) and np.array_equal(order, o2)
        for p in range(cnt.size):
            assert np.array_equal(lst[p, : cnt[p]], l2[p, : c2[p]])


def test_update_then_backward_uses_new_column_view(cuda):
    import torch

    n, d, slots = 640, 64, 2
    a, b = masks_pair(n)
    q, k, v = dev_inputs(cuda, slots, n, d, seed=3)
    g = dev_inputs(cuda, slots, n, d, seed=4)[0]
    scale = 1 / np.sqrt(d)

    def grads(prep):
        o, m, l = fwd(prep, bbm.Variant.binblk, q, k, v)
        dq, dk, dv = (torch.empty_like(q) for _ in range(3))
        bbm.attn_bwd_device(prep, bbm.Variant.binblk, q, k, v, o, m, l, g, dq, dk, dv, scale)
        return dq, dk, dv

    prep = bbm.preprocess_mask(a, bbm.BlockSpec(128, 128))
    grads(prep)  # builds the column view of mask a
    prep.update(torch.from_numpy(b.to_dense()).to(cuda))
    got = grads(prep)
    want = grads(bbm.preprocess_mask(b, bbm.BlockSpec(128, 128)))
    torch.cuda.synchronize()
    assert same(got, want)


def test_update_then_multi_gpu_driver(cuda):
    """run_attention_multi after an update runs the NEW mask on every device (the cached
    replicas are dropped), here over every visible GPU (one on the single-GPU box)."""
    import torch

    n, d, slots = 512, 64, 4
    a, b = masks_pair(n)
    rng = np.random.default_rng(0)
    q, k, v = ((rng.uniform(-1, 1, (slots, n, d)).astype(np.float32)) for _ in range(3))
    qb, kb, vb = (torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16) for x in (q, k, v))
    devices = list(range(torch.cuda.device_count()))
    prep = bbm.preprocess_mask(a, bbm.BlockSpec(128, 128))
    bbm.run_attention_multi(prep, bbm.Variant.binblk, qb, kb, vb, 1 / np.sqrt(d), devices)  # caches replicas
    prep.update(torch.from_numpy(b.to_dense()).to(cuda))
    torch.cuda.synchronize()
    got = bbm.run_attention_multi(prep, bbm.Variant.binblk, qb, kb, vb, 1 / np.sqrt(d), devices)
    want = bbm.run_attention_multi(bbm.preprocess_mask(b, bbm.BlockSpec(128, 128)), bbm.Variant.binblk,
                                   qb, kb, vb, 1 / np.sqrt(d), [0])
    for x, y in zip(got[:3], want[:3]):
        assert np.array_equal(x, y)


@pytest.mark.skipif(not __import__("torch").cuda.is_available() or __import__("torch").cuda.device_count() < 2,
                    reason="needs two GPUs")
def test_two_gpu_driver_equals_one_gpu(cuda):
    import torch

    n, d, slots = 2048, 128, 6
    mask = bbm.gen_longformer_global(n, 200, 64)
    rng = np.random.default_rng(1)
    q, k, v = ((rng.uniform(-1, 1, (slots, n, d)).astype(np.float32)) for _ in range(3))
    qb, kb, vb = (torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16) for x in (q, k, v))
    prep = bbm.preprocess_mask(mask, bbm.BlockSpec(128, 128))
    one = bbm.run_attention_multi(prep, bbm.Variant.binblk, qb, kb, vb, 1 / np.sqrt(d), [0])
    two = bbm.run_attention_multi(prep, bbm.Variant.binblk, qb, kb, vb, 1 / np.sqrt(d), [0, 1])
    for x, y in zip(one[:3], two[:3]):
        assert np.array_equal(x, y)


def test_two_streams_concurrently_on_one_prep(cuda):
    """Launches on two streams sharing one prep overlap and still match the single-stream run
    bitwise (per-stream work counters, plans and split-KV workspace)."""
    import torch

    n, d = 4096, 128
    mask = bbm.gen_longformer_global(n, 300, 128)  # global rows: split-KV units
    prep = bbm.preprocess_mask(mask, bbm.BlockSpec(128, 128))
    ins = [dev_inputs(cuda, 4, n, d, seed=s) for s in (5, 6)]
    want = [fwd(prep, bbm.Variant.binblk, *x) for x in ins]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(cuda) for _ in range(2)]
    outs = [[None] * 2 for _ in range(6)]
    for rep in range(6):
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                outs[rep][i] = fwd(prep, bbm.Variant.binblk, *ins[i], stream=s.cuda_stream)
    torch.cuda.synchronize()
    for rep in range(6):
        for i in range(2):
            assert same(outs[rep][i], want[i])


def _ipc_child(blob, q_path, conn):
    try:
        import torch

        import paper_2409_15097_b200 as b2

        prep = b2.import_prep_ipc(blob, 0)
        arrs = np.load(q_path)
        q, k, v = (torch.from_numpy(arrs[x]).view(torch.bfloat16).cuda() for x in ("q", "k", "v"))
        out = torch.empty_like(q)
        m = torch.empty(q.shape[:2], dtype=torch.float32, device=q.device)
        l = torch.empty_like(m)
        b2.attn_fwd_device(prep, b2.Variant.binblk, q, k, v, out, m, l, 1 / np.sqrt(q.shape[-1]))
        torch.cuda.synchronize()
        conn.send((out.view(torch.int16).cpu().numpy(), m.cpu().numpy(), l.cpu().numpy(),
                   prep.sums.values, prep.counters(b2.Variant.binblk, 2).__dict__))
    except Exception as e:  # noqa: BLE001
        conn.send(repr(e))


def test_ipc_export_import_across_processes(cuda, tmp_path):
    """bench.py's multi-rank path: rank 0 exports, another process imports (here on the same GPU)
    and its forward equals the exporter's bitwise."""
    import torch

    n, d, slots = 1500, 128, 2
    mask = bbm.gen_longformer_global(n, 130, 20)
    prep = bbm.preprocess_mask(mask, bbm.BlockSpec(64, 64))
    q, k, v = dev_inputs(cuda, slots, n, d, seed=9)
    want = fwd(prep, bbm.Variant.binblk, q, k, v)
    torch.cuda.synchronize()
    path = str(tmp_path / "qkv.npz")
    np.savez(path, **{x: t.view(torch.int16).cpu().numpy() for x, t in zip("qkv", (q, k, v))})
    blob = prep.export_ipc()
    ctx = mp.get_context("spawn")
    parent, child = ctx.Pipe()
    p = ctx.Process(target=_ipc_child, args=(blob, path, child))
    p.start()
    got = parent.recv()
    p.join(timeout=120)
    assert not isinstance(got, str), got
    out, m, l, sums, counters = got
    assert np.array_equal(out, want[0].view(torch.int16).cpu().numpy())
    assert np.array_equal(m, want[1].cpu().numpy()) and np.array_equal(l, want[2].cpu().numpy())
    assert np.array_equal(sums, prep.sums.values)
    assert counters == prep.counters(bbm.Variant.binblk, 2).__dict__


def test_run_attention_host_f32_per_slot_equals_device(cuda):
    import torch

    n, d, slots = 700, 64, 3
    mask = bbm.gen_packed_sequential([300, 400])
    prep = bbm.preprocess_mask(mask, bbm.BlockSpec(128, 128))
    q, k, v, _ = oracle.make_problem(11, slots, n, d)
    qf, kf, vf = (np.ascontiguousarray(oracle.bf16_round(x).astype(np.float32)) for x in (q, k, v))
    # one separately allocated Matrix<float> per slot (SlotInputs)
    per = [[np.ascontiguousarray(x[s]) for s in range(slots)] for x in (qf, kf, vf)]
    outs = [np.empty((n, d), np.float32) for _ in range(slots)]
    rms = [np.empty(n, np.float64) for _ in range(slots)]
    rss = [np.empty(n, np.float64) for _ in range(slots)]
    arr = lambda xs: (C.c_void_p * slots)(*[x.ctypes.data for x in xs])  # noqa: E731
    _lib.check(_lib.lib.bbm_run_attention_host_f32(prep.handle.h, int(bbm.Variant.binblk), arr(per[0]),
                                                   arr(per[1]), arr(per[2]), arr(outs), arr(rms), arr(rss),
                                                   slots, d, 1 / np.sqrt(d)))
    dev = [torch.from_numpy(x).to(cuda).to(torch.bfloat16) for x in (qf, kf, vf)]
    o, m, l = fwd(prep, bbm.Variant.binblk, *dev)
    torch.cuda.synchronize()
    for s in range(slots):
        assert np.array_equal(outs[s], o[s].float().cpu().numpy())
        assert np.array_equal(rms[s], m[s].double().cpu().numpy())
        assert np.array_equal(rss[s], l[s].double().cpu().numpy())
    # the contiguous form is the same call
    r = bbm.blocked_forward(qf, kf, vf, 1 / np.sqrt(d), mask, prep, bbm.Variant.binblk)
    assert np.array_equal(r.out, np.stack(outs))


@pytest.mark.parametrize("which", ["f32", "bf16"])
def test_host_paths_reject_non_finite(cuda, which):
    import torch

    n, d, slots = 256, 64, 2
    mask = bbm.gen_causal(n)
    prep = bbm.preprocess_mask(mask, bbm.BlockSpec(128, 128))
    q, k, v, _ = oracle.make_problem(3, slots, n, d)
    q, k, v = (x.astype(np.float32) for x in (q, k, v))
    v[1, 7, 3] = np.nan
    if which == "f32":
        with pytest.raises(ValueError, match="v must hold finite values"):
            bbm.blocked_forward(q, k, v, 0.125, mask, prep, bbm.Variant.binblk)
    else:
        qb, kb, vb = (torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
                      for x in (q, k, v))
        out = np.empty_like(qb)
        u16 = C.POINTER(C.c_uint16)
        st = _lib.lib.bbm_attn_fwd_host_bf16(prep.handle.h, 2, qb.ctypes.data_as(u16), kb.ctypes.data_as(u16),
                                             vb.ctypes.data_as(u16), out.ctypes.data_as(u16), None, None,
                                             slots, d, 0.125)
        assert st == _lib.BBM_ERR_INVALID and b"v must hold finite" in _lib.lib.bbm_last_error()


def test_device_entry_rejects_mismatched_shapes(cuda):
    """k/v with fewer slots than q must be rejected before any TMA descriptor covers
    memory that does not exist."""
    import torch

    n, d = 256, 64
    mask = bbm.gen_causal(n)
    prep = bbm.preprocess_mask(mask, bbm.BlockSpec(128, 128))
    q = torch.zeros((3, n, d), dtype=torch.bfloat16, device=cuda)
    k = torch.zeros((n, d), dtype=torch.bfloat16, device=cuda)
    with pytest.raises(ValueError):
        bbm.blocked_forward(q, k, k, 0.125, mask, prep, bbm.Variant.binblk)
    with pytest.raises(ValueError):
        bbm.attn_fwd_device(prep, bbm.Variant.binblk, q, k.expand(3, n, d), q, torch.empty_like(q))
    with pytest.raises(ValueError, match="scale"):
        bbm.blocked_forward(q, q, q, 1e39, mask, prep, bbm.Variant.binblk)
    # a contiguous view 2 bytes into its storage: rejected before any TMA descriptor / cp.async
    buf = torch.zeros(3 * n * d + 8, dtype=torch.bfloat16, device=cuda)
    mis = buf[1:1 + 3 * n * d].view(3, n, d)
    rows = torch.arange(n, dtype=torch.int32, device=cuda)
    for kw in ({}, {"rows": rows, "gather_mode": 4}, {"rows": rows, "gather_mode": 2}):
        with pytest.raises(ValueError, match="aligned"):
            bbm.attn_fwd_device(prep, bbm.Variant.binblk, mis, q, q, torch.empty_like(q), **kw)


@pytest.mark.parametrize("pinned", [False, True])
def test_float_host_path_rounding_equals_device(cuda, pinned):
    """The float host path converts part of the slots on the host (all of them for pageable
    buffers, ~70 % for pinned ones) and the rest on the device: both must round to nearest even
    exactly like torch's device conversion, on values that are NOT bf16-representable."""
    import torch

    n, d, slots = 900, 128, 7
    mask = bbm.gen_longformer_windowed(n, 60)
    prep = bbm.preprocess_mask(mask, bbm.BlockSpec(128, 128))
    g = torch.Generator().manual_seed(5)
    host = [torch.rand((slots, n, d), generator=g) * 6 - 3 for _ in range(3)]
    if pinned:
        host = [t.pin_memory() for t in host]
    outs = torch.empty((slots, n, d), dtype=torch.float32)
    rms = torch.empty((slots, n), dtype=torch.float64)
    rss = torch.empty((slots, n), dtype=torch.float64)
    if pinned:
        outs, rms, rss = outs.pin_memory(), rms.pin_memory(), rss.pin_memory()
    arr = lambda t: (C.c_void_p * slots)(*[t[s].data_ptr() for s in range(slots)])  # noqa: E731
    _lib.check(_lib.lib.bbm_run_attention_host_f32(prep.handle.h, int(bbm.Variant.binblk), arr(host[0]),
                                                   arr(host[1]), arr(host[2]), arr(outs), arr(rms), arr(rss),
                                                   slots, d, 0.07))
    dev = [t.to(cuda).to(torch.bfloat16) for t in host]
    o, m, l = fwd(prep, bbm.Variant.binblk, *dev, scale=0.07)
    torch.cuda.synchronize()
    assert torch.equal(outs, o.float().cpu())
    assert torch.equal(rms, m.double().cpu()) and torch.equal(rss, l.double().cpu())
