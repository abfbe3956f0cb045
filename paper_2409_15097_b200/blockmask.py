"""Python mirror of the reference's C++ API (namespace blockmask, /root/reference/proj/include).

Same names, argument meaning and error behaviour as the reference headers, so callers and tests
read like the reference's own; every compute call goes through libbbm.so's C ABI to the sm_100a
kernels. ``ValueError`` plays the role of ``std::invalid_argument``.

  reference (file:line)                      here
  Mask (mask.hpp:17-52)                      Mask           packed u64 words, same layout
  BlockSpec (mask.hpp:57-66)                 BlockSpec
  BlockSums / BlockOccupancy / DenseRuns /   BlockSums / BlockOccupancy / DenseRuns / BlockStats
    BlockStats (mask.hpp:71-162)
  block_sums, build_block_occupancy,         same names; computed by the GPU preprocessor
    build_dense_runs, block_stats (:184-247)
  Variant, to_string, parse_variant          same
    (engine.hpp:21-45)
  EngineCounters (engine.hpp:49-66)          EngineCounters
  MaskPrep, preprocess_mask (:71-91)         MaskPrep, preprocess_mask  (+ device metadata)
  ForwardResult (engine.hpp:93-99)           ForwardResult
  blocked_forward (engine.hpp:282-341)       blocked_forward   (torch CUDA bf16 or host float)
  SlotInputs / MultiHeadForward /            SlotInputs / MultiHeadForward / run_attention
    run_attention (engine.hpp:475-505)
  rcm_order / bandwidth / permute_rows /     rcm_order / bandwidth / permute_rows /
    unpermute_rows / permute_mask              unpermute_rows / permute_mask (reorder.hpp)
  generators (generators.hpp)                gen_* / generate
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import Iterable, List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import check, lib, ptr

# ----------------------------------------------------------------------------- mask model


@dataclass(frozen=True)
class BlockSpec:
    """Tile shape (mask.hpp:57-66); default 64 x 64 like the reference."""
    block_i: int = 64
    block_j: int = 64

    def validate(self) -> None:
        if self.block_i < 1 or self.block_j < 1:
            raise ValueError("block sizes must be >= 1")


class Mask:
    """Square bit-packed attention mask, the reference's layout (mask.hpp:17-52):
    row-major u64 words, words_per_row = ceil(n/64), bit j of row i at word j>>6 bit j&63,
    tail bits zero."""

    def __init__(self, n: int = 0, words: Optional[np.ndarray] = None):
        self._n = int(n)
        self._wpr = (self._n + 63) // 64
        if words is None:
            self.words = np.zeros((self._n, self._wpr), dtype=np.uint64)
        else:
            w = np.ascontiguousarray(words, dtype=np.uint64).reshape(self._n, self._wpr)
            self.words = w

    def size(self) -> int:
        return self._n

    def words_per_row(self) -> int:
        return self._wpr

    def get(self, i: int, j: int) -> bool:
        return bool((int(self.words[i, j >> 6]) >> (j & 63)) & 1)

    def set(self, i: int, j: int, value: bool) -> None:
        bit = np.uint64(1 << (j & 63))
        if value:
            self.words[i, j >> 6] |= bit
        else:
            self.words[i, j >> 6] &= ~bit

    def row_words(self, i: int) -> np.ndarray:
        return self.words[i]

    def count_ones(self) -> int:
        return int(np.unpackbits(self.words.view(np.uint8)).sum())

    def to_dense(self) -> np.ndarray:
        bits = np.unpackbits(self.words.view(np.uint8), axis=1, bitorder="little")
        return bits[:, : self._n].astype(bool)

    @staticmethod
    def from_dense(dense: np.ndarray) -> "Mask":
        dense = np.asarray(dense, dtype=bool)
        n = dense.shape[0]
        if dense.shape != (n, n):
            raise ValueError("mask must be square")
        wpr = (n + 63) // 64
        pad = np.zeros((n, wpr * 64), dtype=np.uint8)
        pad[:, :n] = dense
        packed = np.packbits(pad, axis=1, bitorder="little")
        return Mask(n, packed.view(np.uint64).reshape(n, wpr))

    def __eq__(self, other) -> bool:
        return isinstance(other, Mask) and self._n == other._n and np.array_equal(self.words, other.words)


class BlockSums:
    """Per-block one counts with edge geometry (mask.hpp:71-109)."""

    def __init__(self, n_tokens: int, spec: BlockSpec, sums: np.ndarray):
        self._n = n_tokens
        self._spec = spec
        self.values = sums

    def n_tokens(self) -> int:
        return self._n

    def spec(self) -> BlockSpec:
        return self._spec

    def rows(self) -> int:
        return self.values.shape[0]

    def cols(self) -> int:
        return self.values.shape[1]

    def sum(self, p: int, q: int) -> int:
        return int(self.values[p, q])

    def rows_in_block(self, p: int) -> int:
        return min(self._spec.block_i, self._n - p * self._spec.block_i)

    def cols_in_block(self, q: int) -> int:
        return min(self._spec.block_j, self._n - q * self._spec.block_j)

    def block_area(self, p: int, q: int) -> int:
        return self.rows_in_block(p) * self.cols_in_block(q)

    def full(self, p: int, q: int) -> bool:
        return self.sum(p, q) == self.block_area(p, q)


class BlockOccupancy:
    """u8 per block, 1 iff any set bit (mask.hpp:113-132)."""

    def __init__(self, occ: np.ndarray):
        self.values = occ

    def rows(self) -> int:
        return self.values.shape[0]

    def cols(self) -> int:
        return self.values.shape[1]

    def at(self, p: int, q: int) -> bool:
        return bool(self.values[p, q])

    def __eq__(self, other) -> bool:
        return isinstance(other, BlockOccupancy) and np.array_equal(self.values, other.values)


@dataclass
class DenseRuns:
    """First maximal run of full blocks per row block (mask.hpp:139-154), half-open."""
    offset: List[int]
    total_ones: List[int]

    def in_run(self, r: int, q: int) -> bool:
        return self.offset[r] <= q < self.offset[r] + self.total_ones[r]

    def total_run_blocks(self) -> int:
        return int(sum(self.total_ones))


@dataclass
class BlockStats:
    blocks_total: int = 0
    blocks_nonzero: int = 0
    blocks_full: int = 0
    block_density: float = 0.0
    element_density: float = 0.0


@dataclass
class EngineCounters:
    """Deterministic tile bookkeeping (engine.hpp:49-66)."""
    blocks_visited: int = 0
    blocks_processed: int = 0
    mask_block_reads: int = 0
    skipped_by_binblk: int = 0
    skipped_mask_reads_by_run: int = 0

    def __iadd__(self, o: "EngineCounters") -> "EngineCounters":
        self.blocks_visited += o.blocks_visited
        self.blocks_processed += o.blocks_processed
        self.mask_block_reads += o.mask_block_reads
        self.skipped_by_binblk += o.skipped_by_binblk
        self.skipped_mask_reads_by_run += o.skipped_mask_reads_by_run
        return self


class Variant(enum.IntEnum):
    """engine.hpp:21-26"""
    dense = 0
    naive_masked = 1
    binblk = 2
    dense_binblk = 3


_VARIANT_NAMES = {Variant.dense: "dense", Variant.naive_masked: "naive", Variant.binblk: "binblk",
                  Variant.dense_binblk: "dense-binblk"}


def to_string(v: Variant) -> str:
    return _VARIANT_NAMES.get(Variant(v), "?")


def parse_variant(name: str) -> Variant:
    for v, s in _VARIANT_NAMES.items():
        if s == name:
            return v
    raise ValueError(f"unknown variant: '{name}' (expected dense, naive, binblk, dense-binblk)")


# ----------------------------------------------------------------------------- preprocessing


class _PrepHandle:
    """Owns a bbm_prep (device metadata); destroyed with the Python object."""

    def __init__(self, h: C.c_void_p):
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            lib.bbm_prep_destroy(self.h)
            self.h = None


class MaskPrep:
    """engine.hpp:71-78 plus the device-resident kernel metadata (``handle``).

    The host-side fields (``sums``, ``occupancy``, ``runs``, ``stats``) are read from the C ABI,
    which recomputes them after :meth:`update` (a new mask of the same size, rebuilt on the device
    without a host round trip); they are cached per update."""

    def __init__(self, handle: _PrepHandle):
        self.handle = handle
        self._version = 0
        self._cache = {}
        info = self.info()
        self.n_tokens = int(info.n)
        self.spec = BlockSpec(int(info.block_i), int(info.block_j))

    def __repr__(self) -> str:
        return f"MaskPrep(n_tokens={self.n_tokens}, spec={self.spec})"

    def _host(self):
        got = self._cache.get(self._version)
        if got is None:
            h = self.handle.h
            info = self.info()
            rows, cols = int(info.rows), int(info.cols)
            sums = np.zeros((rows, cols), np.uint32)
            occ = np.zeros((rows, cols), np.uint8)
            off = np.zeros(rows, np.uint32)
            tot = np.zeros(rows, np.uint32)
            st = _lib.BlockStatsC()
            check(lib.bbm_prep_get_sums(h, ptr(sums, C.c_uint32)))
            check(lib.bbm_prep_get_occupancy(h, ptr(occ, C.c_uint8)))
            check(lib.bbm_prep_get_runs(h, ptr(off, C.c_uint32), ptr(tot, C.c_uint32)))
            check(lib.bbm_prep_get_stats(h, C.byref(st)))
            got = (BlockSums(self.n_tokens, self.spec, sums), BlockOccupancy(occ),
                   DenseRuns([int(x) for x in off], [int(x) for x in tot]),
                   BlockStats(st.blocks_total, st.blocks_nonzero, st.blocks_full, st.block_density,
                              st.element_density))
            self._cache = {self._version: got}
        return got

    @property
    def sums(self) -> BlockSums:
        return self._host()[0]

    @property
    def occupancy(self) -> BlockOccupancy:
        return self._host()[1]

    @property
    def runs(self) -> DenseRuns:
        return self._host()[2]

    @property
    def stats(self) -> BlockStats:
        return self._host()[3]

    def info(self) -> _lib.PrepInfoC:
        info = _lib.PrepInfoC()
        check(lib.bbm_prep_get_info(self.handle.h, C.byref(info)))
        return info

    def kernel_lists(self):
        """(row_cnt[krows], list[krows, kcols] with bit 31 = full, LPT order[krows])."""
        info = self.info()
        cnt = np.zeros(info.krows, np.uint32)
        lst = np.zeros((info.krows, info.kcols), np.uint32)
        order = np.zeros(info.krows, np.uint32)
        check(lib.bbm_prep_get_kernel_lists(self.handle.h, ptr(cnt, C.c_uint32), ptr(lst, C.c_uint32),
                                            ptr(order, C.c_uint32)))
        return cnt, lst, order

    def tile_halves(self):
        """u8 [krows, kcols] at list positions: bit 0 / 1 = key columns 0-63 / 64-127 of the
        occupied tile empty for all its rows (the forward skips that half)."""
        info = self.info()
        h = np.zeros((info.krows, info.kcols), np.uint8)
        check(lib.bbm_prep_get_tile_halves(self.handle.h, ptr(h, C.c_uint8)))
        return h

    def counters(self, variant: Variant, slots: int = 1) -> EngineCounters:
        c = _lib.CountersC()
        check(lib.bbm_prep_counters(self.handle.h, int(variant), int(slots), C.byref(c)))
        return EngineCounters(c.blocks_visited, c.blocks_processed, c.mask_block_reads,
                              c.skipped_by_binblk, c.skipped_mask_reads_by_run)

    def update(self, mask, stream=None) -> None:
        """Rebuild for a new mask of the same size, asynchronously on ``stream`` (a CUDA
        ``torch.bool``/``uint8`` n x n tensor, or ``torch.int64`` packed words [n][ceil(n/64)])."""
        import torch

        if not isinstance(mask, torch.Tensor) or not mask.is_cuda or mask.shape[0] != self.n_tokens:
            raise ValueError("update needs a CUDA mask tensor of the prep's size")
        s = stream if stream is not None else torch.cuda.current_stream(mask.device).cuda_stream
        with torch.cuda.device(mask.device):
            if mask.dtype in (torch.bool, torch.uint8):
                m = mask if mask.stride(1) == 1 else mask.contiguous()
                check(lib.bbm_prep_update_bool_device(self.handle.h, C.c_void_p(m.data_ptr()), m.stride(0),
                                                      C.c_void_p(s)))
            elif mask.dtype == torch.int64:
                m = mask.contiguous()
                check(lib.bbm_prep_update_packed_device(self.handle.h, C.c_void_p(m.data_ptr()), C.c_void_p(s)))
            else:
                raise ValueError("unsupported mask tensor dtype")
        self._version += 1

    def replicate(self, device: int) -> "MaskPrep":
        """bbm_prep_replicate: the same metadata on another GPU (peer-to-peer copy)."""
        h = C.c_void_p()
        check(lib.bbm_prep_replicate(self.handle.h, int(device), None, C.byref(h)))
        return MaskPrep(_PrepHandle(h))

    def export_ipc(self) -> bytes:
        """bbm_prep_export_ipc: a blob another process imports with :func:`import_prep_ipc`."""
        size = C.c_size_t(0)
        check(lib.bbm_prep_export_ipc(self.handle.h, None, C.byref(size)))
        buf = (C.c_uint8 * size.value)()
        check(lib.bbm_prep_export_ipc(self.handle.h, C.cast(buf, C.c_void_p), C.byref(size)))
        return bytes(buf)


def import_prep_ipc(blob: bytes, device: int = 0) -> MaskPrep:
    """bbm_prep_import_ipc: copy an exported prep's device metadata (IPC + peer copy) onto
    ``device`` of this process."""
    h = C.c_void_p()
    buf = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
    check(lib.bbm_prep_import_ipc(C.cast(buf, C.c_void_p), len(blob), int(device), None, C.byref(h)))
    return MaskPrep(_PrepHandle(h))


def _prep_from_handle(h: C.c_void_p) -> MaskPrep:
    return MaskPrep(_PrepHandle(h))


def preprocess_mask(mask, spec: BlockSpec = BlockSpec(), device: int = 0, stream=None) -> MaskPrep:
    """preprocess_mask (engine.hpp:80-91) on the GPU.

    ``mask`` may be a :class:`Mask` (host, bit-packed), a CUDA ``torch.bool``/``uint8`` n x n
    tensor (dense mask: K1 pack + sums kernel) or a CUDA ``torch.int64`` tensor holding the packed
    words [n][ceil(n/64)].
    """
    spec.validate()
    h = C.c_void_p()
    if isinstance(mask, Mask):
        if mask.size() < 1:
            raise ValueError("mask must be non-empty")
        words = np.ascontiguousarray(mask.words)
        check(lib.bbm_preprocess_packed_host(ptr(words, C.c_uint64), mask.size(), spec.block_i,
                                             spec.block_j, device, C.byref(h)))
        return _prep_from_handle(h)
    import torch  # device path

    if not isinstance(mask, torch.Tensor) or not mask.is_cuda:
        raise ValueError("mask must be a Mask or a CUDA tensor")
    s = stream if stream is not None else torch.cuda.current_stream(mask.device).cuda_stream
    with torch.cuda.device(mask.device):
        if mask.dtype in (torch.bool, torch.uint8):
            n = mask.shape[0]
            if mask.dim() != 2 or mask.shape[1] != n:
                raise ValueError("dense mask must be n x n")
            m = mask if mask.stride(1) == 1 else mask.contiguous()
            check(lib.bbm_preprocess_bool_device(C.c_void_p(m.data_ptr()), n, m.stride(0),
                                                 spec.block_i, spec.block_j, C.c_void_p(s), C.byref(h)))
        elif mask.dtype == torch.int64:
            n = mask.shape[0]
            m = mask.contiguous()
            check(lib.bbm_preprocess_packed_device(C.c_void_p(m.data_ptr()), n, spec.block_i,
                                                   spec.block_j, C.c_void_p(s), C.byref(h)))
        else:
            raise ValueError("unsupported mask tensor dtype")
    return _prep_from_handle(h)


def block_sums(mask, spec: BlockSpec) -> BlockSums:
    """block_sums (mask.hpp:184-201), computed by the GPU preprocessor."""
    return preprocess_mask(mask, spec).sums


def _sums_metadata(sums: BlockSums, device: int = 0):
    """build_block_occupancy + build_dense_runs + block_stats of caller-held sums, computed by
    the preprocessor's per-row-tile kernel on the GPU (C ABI bbm_sums_metadata)."""
    spec = sums.spec()
    vals = np.ascontiguousarray(sums.values, dtype=np.uint32)
    occ = np.empty(vals.shape, np.uint8)
    off = np.empty(sums.rows(), np.uint32)
    tot = np.empty(sums.rows(), np.uint32)
    st = _lib.BlockStatsC()
    check(lib.bbm_sums_metadata(ptr(vals, C.c_uint32), sums.n_tokens(), spec.block_i, spec.block_j, device,
                                ptr(occ, C.c_uint8), ptr(off, C.c_uint32), ptr(tot, C.c_uint32), C.byref(st)))
    return occ, off, tot, st


def build_block_occupancy(sums: BlockSums) -> BlockOccupancy:
    """build_block_occupancy (mask.hpp:203-209), on the GPU."""
    return BlockOccupancy(_sums_metadata(sums)[0])


def build_dense_runs(sums: BlockSums) -> DenseRuns:
    """build_dense_runs (mask.hpp:213-228), on the GPU."""
    _, off, tot, _ = _sums_metadata(sums)
    return DenseRuns(off.tolist(), tot.tolist())


def block_stats(sums: BlockSums) -> BlockStats:
    """block_stats (mask.hpp:230-247), on the GPU."""
    st = _sums_metadata(sums)[3]
    return BlockStats(int(st.blocks_total), int(st.blocks_nonzero), int(st.blocks_full),
                      float(st.block_density), float(st.element_density))


# ----------------------------------------------------------------------------- attention


@dataclass
class ForwardResult:
    """engine.hpp:93-99. ``out`` keeps the input's container type; row stats as float64."""
    out: object
    row_max: object
    row_sum: object
    counters: EngineCounters


@dataclass
class SlotInputs:
    q: object
    k: object
    v: object


@dataclass
class MultiHeadForward:
    slots: List[ForwardResult]
    counters: EngineCounters


def _validate_common(prep: MaskPrep, mask, scale: float, threads: int) -> None:
    # validate_forward_args (engine.hpp:244-258)
    n = mask.size() if isinstance(mask, Mask) else int(mask.shape[0])
    if prep.n_tokens != n:
        raise ValueError("mask preprocessing does not match this mask")
    if not math.isfinite(scale):
        raise ValueError("scale must be finite")
    if threads < 1:
        raise ValueError("thread count must be >= 1")


def attn_fwd_device(prep: MaskPrep, variant: Variant, q, k, v, out, row_max=None, row_sum=None,
                    scale: float = 1.0, stream=None, rows=None, gather_mode: int = 0) -> None:
    """Raw launch on device tensors (bf16 [slots][n][d], contiguous). No validation beyond
    shapes; this is the timed entry point. row_max / row_sum: float32 [slots][n] or None.

    ``rows``: optional CUDA int32/uint32 tensor [n], an RCM permutation's forward map (new -> old)
    for a prep built from ``permute_mask(mask, perm)``: the tensors then stay in the ORIGINAL
    token order and the RCM permutation is applied on the device (bbm_attn_fwd_gather_ex):
    ``gather_mode`` 0 = the default, the fastest on B200 (4), 1 = permute / unpermute passes around the
    plain kernel, 2 = in-kernel TMA tile::gather4 / scatter4, 3 = K / V permuted by passes with
    Q rows gathered and O rows scattered in the kernel, 4 = every row gathered in the kernel by
    LSU cp.async (no scratch)."""
    import torch

    slots, n, d = (q.shape if q.dim() == 3 else (1, *q.shape))
    for t in (k, v, out):
        if t.shape != q.shape or not t.is_contiguous() or t.dtype != torch.bfloat16:
            raise ValueError("q, k, v, out must be contiguous bf16 tensors of one shape")
    for t in (row_max, row_sum):
        if t is not None and (t.numel() != slots * n or t.dtype != torch.float32):
            raise ValueError("row statistics must be float32 [slots][n]")
    s = stream if stream is not None else torch.cuda.current_stream(q.device).cuda_stream
    if rows is not None:
        if rows.numel() != n or rows.element_size() != 4 or not rows.is_cuda or not rows.is_contiguous():
            raise ValueError("rows must be a contiguous CUDA 32-bit tensor of n entries")
        check(lib.bbm_attn_fwd_gather_ex(prep.handle.h, int(variant), C.c_void_p(rows.data_ptr()),
                                      C.c_void_p(q.data_ptr()), C.c_void_p(k.data_ptr()), C.c_void_p(v.data_ptr()),
                                      C.c_void_p(out.data_ptr()),
                                      C.c_void_p(row_max.data_ptr() if row_max is not None else 0),
                                      C.c_void_p(row_sum.data_ptr() if row_sum is not None else 0),
                                      int(slots), int(d), float(scale), C.c_void_p(s), int(gather_mode)))
        return
    check(lib.bbm_attn_fwd(prep.handle.h, int(variant), C.c_void_p(q.data_ptr()), C.c_void_p(k.data_ptr()),
                           C.c_void_p(v.data_ptr()), C.c_void_p(out.data_ptr()),
                           C.c_void_p(row_max.data_ptr() if row_max is not None else 0),
                           C.c_void_p(row_sum.data_ptr() if row_sum is not None else 0),
                           int(slots), int(d), float(scale), C.c_void_p(s)))


def set_fwd_kernel(mode: str) -> None:
    """Forward kernel selection (bbm_set_fwd_kernel): "auto" / "single" (attn_fwd.cu, the default)
    or "pair" (attn_fwd_pair.cu wherever it can run; measured slower, kept for comparison)."""
    modes = {"auto": 0, "single": 1, "pair": 2}
    if mode not in modes:
        raise ValueError(f"unknown forward kernel mode {mode!r}")
    check(lib.bbm_set_fwd_kernel(modes[mode]))


def _check_head_dims(dk: int, dv: int) -> None:
    """validate_forward_args (engine.hpp:249-251) plus the documented narrowing d_k <= 128."""
    if dk < 1:
        raise ValueError("q and k must share a positive head dim")
    if dv < 1:
        raise ValueError("v must have a positive head dim")
    if dk > 128:
        raise ValueError(f"head dim d_k = {dk} unsupported by the sm_100a kernel (at most 128)")


def _kernel_dim(dk: int, dv: int) -> int:
    """The kernels' head dim for caller dims d_k, d_v (bbm_internal.h kernel_dim)."""
    return 128 if max(dk, dv) > 64 else 64


def _pad_cols(t, D: int):
    """Zero-pad the last dim to D: zero Q/K columns add exact zeros to every score, zero V / dO
    columns give output columns that are cropped away."""
    if t.shape[-1] == D:
        return t
    import torch.nn.functional as F
    return F.pad(t, (0, D - t.shape[-1]))


def blocked_forward(q, k, v, scale: float, mask, prep: MaskPrep, variant: Variant,
                    threads: int = 1, check_finite: bool = True) -> ForwardResult:
    """blocked_forward (engine.hpp:282-341) on the sm_100a kernel.

    q, k, v: CUDA bf16 tensors [n, d] or [slots, n, d] (device path, result stays on device), or
    numpy float arrays [n, d] (host path, like Matrix<float>; rounded to bf16 on the device).
    Head dims d_k (q, k) and d_v (v, out) may differ; d_k at most 128 (documented narrowing: the
    kernels hold one 128-column head-dim tile). Dims other than 64 / 128 run zero-padded, d_v above
    128 as column passes over V."""
    _validate_common(prep, mask, scale, threads)
    n = prep.n_tokens
    if isinstance(q, np.ndarray):
        return _blocked_forward_host(q, k, v, scale, prep, variant)
    import torch

    if q.shape[-2] != n or k.shape[-2] != n or v.shape[-2] != n:
        raise ValueError("q/k/v row count must match mask size")
    if q.shape[-1] != k.shape[-1] or q.shape[-1] < 1:
        raise ValueError("q and k must share a positive head dim")
    if v.shape[-1] < 1:
        raise ValueError("v must have a positive head dim")
    if q.shape != k.shape or q.shape[:-1] != v.shape[:-1] or q.dim() not in (2, 3):
        raise ValueError("q, k and v must share one [n, d] or [slots, n, d] shape (v may differ in d)")
    _check_head_dims(q.shape[-1], v.shape[-1])
    if not (q.device == k.device == v.device) or not q.is_cuda:
        raise ValueError("q, k and v must live on one CUDA device")
    if check_finite:
        for name, t in (("q", q), ("k", k), ("v", v)):
            if not bool(torch.isfinite(t).all()):
                raise ValueError(f"{name} must hold finite values")
    squeeze = q.dim() == 2
    q3, k3, v3 = (t.unsqueeze(0) if squeeze else t for t in (q, k, v))
    dv = v3.shape[-1]
    slots = q3.shape[0]
    rmax = torch.empty((slots, n), dtype=torch.float32, device=q3.device)
    rsum = torch.empty((slots, n), dtype=torch.float32, device=q3.device)
    parts = []
    for c0 in range(0, dv, 128):  # d_v > 128: column passes over V (capi.cu v_slices)
        w = min(128, dv - c0)
        D = _kernel_dim(q3.shape[-1], w)
        qp, kp, vp = (_pad_cols(t.to(torch.bfloat16), D).contiguous() for t in (q3, k3, v3[..., c0:c0 + w]))
        o = torch.empty_like(vp)
        with torch.cuda.device(q3.device):
            attn_fwd_device(prep, variant, qp, kp, vp, o, rmax, rsum, scale)
        parts.append(o[..., :w])
    out = parts[0].contiguous() if len(parts) == 1 else torch.cat(parts, dim=-1)
    counters = prep.counters(variant, slots)
    if squeeze:
        out, rmax, rsum = out[0], rmax[0], rsum[0]
    return ForwardResult(out, rmax.double(), rsum.double(), counters)


def _blocked_forward_host(q, k, v, scale, prep, variant) -> ForwardResult:
    n = prep.n_tokens
    arrs = [np.ascontiguousarray(a, dtype=np.float32) for a in (q, k, v)]
    squeeze = arrs[0].ndim == 2
    if squeeze:
        arrs = [a[None] for a in arrs]
    qa, ka, va = arrs
    if qa.shape[1] != n or ka.shape[1] != n or va.shape[1] != n:
        raise ValueError("q/k/v row count must match mask size")
    if qa.shape[2] != ka.shape[2] or qa.shape[2] < 1:
        raise ValueError("q and k must share a positive head dim")
    if va.shape[2] < 1:
        raise ValueError("v must have a positive head dim")
    if not (qa.shape[0] == ka.shape[0] == va.shape[0]):
        raise ValueError("q, k and v must hold the same number of slots")
    slots, _, dk = qa.shape
    dv = va.shape[2]
    _check_head_dims(dk, dv)
    out = np.empty((slots, n, dv), np.float32)
    rmax = np.empty((slots, n), np.float64)
    rsum = np.empty((slots, n), np.float64)
    # per-slot pointers (run_attention's storage, engine.hpp:489-505)
    vpa = lambda a, w: (C.c_void_p * slots)(*[a.ctypes.data + i * n * w * a.itemsize for i in range(slots)])  # noqa: E731
    check(lib.bbm_run_attention_host_f32_dims(prep.handle.h, int(variant), vpa(qa, dk), vpa(ka, dk), vpa(va, dv),
                                              vpa(out, dv), vpa(rmax, 1), vpa(rsum, 1), slots, dk, dv,
                                              float(scale)))
    counters = prep.counters(variant, slots)
    if squeeze:
        out, rmax, rsum = out[0], rmax[0], rsum[0]
    return ForwardResult(out, rmax, rsum, counters)


@dataclass
class BackwardResult:
    """engine.hpp:101-107."""
    dq: object
    dk: object
    dv: object
    counters: EngineCounters


def attn_bwd_device(prep: MaskPrep, variant: Variant, q, k, v, out, row_max, row_sum, d_out,
                    dq, dk, dv, scale: float = 1.0, stream=None) -> None:
    """Raw backward launch on device tensors: bf16 [slots][n][d] (q, k, v, out, d_out, dq, dk, dv)
    and float32 [slots][n] row stats as the forward returns them. The timed entry point."""
    import torch

    slots, n, d = (q.shape if q.dim() == 3 else (1, *q.shape))
    s = stream if stream is not None else torch.cuda.current_stream(q.device).cuda_stream
    vp_ = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    check(lib.bbm_attn_bwd(prep.handle.h, int(variant), vp_(q), vp_(k), vp_(v), vp_(out), vp_(row_max),
                           vp_(row_sum), vp_(d_out), vp_(dq), vp_(dk), vp_(dv), int(slots), int(d),
                           float(scale), C.c_void_p(s)))


def blocked_backward(q, k, v, scale: float, mask, prep: MaskPrep, variant: Variant, fwd: ForwardResult,
                     d_out, threads: int = 1) -> BackwardResult:
    """blocked_backward (engine.hpp:346-471) on the sm_100a kernels: gradients of
    L = sum(out * d_out) from the forward's saved row statistics. Same containers as
    blocked_forward (CUDA bf16 tensors or numpy float arrays); counters equal the forward's."""
    _validate_common(prep, mask, scale, threads)
    n = prep.n_tokens
    if isinstance(q, np.ndarray):
        arrs = [np.ascontiguousarray(a, dtype=np.float32) for a in (q, k, v, fwd.out, d_out)]
        squeeze = arrs[0].ndim == 2
        if squeeze:
            arrs = [a[None] for a in arrs]
        qa, ka, va, oa, ga = arrs
        slots, _, dk = qa.shape
        dv = va.shape[2]
        if ka.shape != qa.shape or oa.shape != va.shape or ga.shape != va.shape or va.shape[:2] != qa.shape[:2]:
            raise ValueError("q, k must share [slots][n][d_k]; v, out, d_out [slots][n][d_v]")
        if qa.shape[1] != n:
            raise ValueError("q/k/v row count must match mask size")
        _check_head_dims(dk, dv)
        rm = np.ascontiguousarray(np.asarray(fwd.row_max, np.float64).reshape(slots, n))
        rs = np.ascontiguousarray(np.asarray(fwd.row_sum, np.float64).reshape(slots, n))
        gq, gk, gv = np.empty_like(qa), np.empty_like(ka), np.empty_like(va)
        check(lib.bbm_attn_bwd_host_f32_dims(prep.handle.h, int(variant), ptr(qa, C.c_float), ptr(ka, C.c_float),
                                             ptr(va, C.c_float), ptr(oa, C.c_float), ptr(rm, C.c_double),
                                             ptr(rs, C.c_double), ptr(ga, C.c_float), ptr(gq, C.c_float),
                                             ptr(gk, C.c_float), ptr(gv, C.c_float), slots, dk, dv, float(scale)))
        if squeeze:
            gq, gk, gv = gq[0], gk[0], gv[0]
        return BackwardResult(gq, gk, gv, prep.counters(variant, slots))
    import torch

    squeeze = q.dim() == 2
    ts = [t.unsqueeze(0) if squeeze else t for t in (q, k, v, fwd.out, d_out)]
    if (ts[0].shape != ts[1].shape or len({tuple(t.shape) for t in ts[2:]}) != 1
            or ts[2].shape[:2] != ts[0].shape[:2] or ts[0].shape[1] != n):
        raise ValueError("q, k must share [slots][n][d_k]; v, out, d_out [slots][n][d_v]")
    dk_, dv_ = ts[0].shape[-1], ts[2].shape[-1]
    _check_head_dims(dk_, dv_)
    if dv_ > 128:  # column passes over V: dq, dk summed over the slices, dv concatenated
        fq, fk, fv = None, None, []
        for c0 in range(0, dv_, 128):
            w = min(128, dv_ - c0)
            sl = lambda t: t[..., c0:c0 + w]  # noqa: E731
            part = blocked_backward(q, k, sl(v), scale, mask, prep, variant,
                                    ForwardResult(sl(fwd.out), fwd.row_max, fwd.row_sum, fwd.counters), sl(d_out),
                                    threads)
            fq = part.dq.float() if fq is None else fq + part.dq.float()
            fk = part.dk.float() if fk is None else fk + part.dk.float()
            fv.append(part.dv)
        return BackwardResult(fq.to(torch.bfloat16), fk.to(torch.bfloat16), torch.cat(fv, dim=-1),
                              prep.counters(variant, ts[0].shape[0]))
    D = _kernel_dim(dk_, dv_)
    for name, t in (("q", q), ("k", k), ("v", v), ("d_out", d_out)):
        if not bool(torch.isfinite(t).all()):
            raise ValueError(f"{name} must hold finite values")
    q3, k3, v3, o3, g3 = (_pad_cols(t.to(torch.bfloat16), D).contiguous() for t in ts)
    slots = q3.shape[0]
    rm = torch.as_tensor(fwd.row_max, device=q3.device).reshape(slots, n).float().contiguous()
    rs = torch.as_tensor(fwd.row_sum, device=q3.device).reshape(slots, n).float().contiguous()
    dq, dk, dv = (torch.empty_like(q3) for _ in range(3))
    with torch.cuda.device(q3.device):
        attn_bwd_device(prep, variant, q3, k3, v3, o3, rm, rs, g3, dq, dk, dv, scale)
    if D != dk_:
        dq, dk = dq[..., :dk_].contiguous(), dk[..., :dk_].contiguous()
    if D != dv_:
        dv = dv[..., :dv_].contiguous()
    if squeeze:
        dq, dk, dv = dq[0], dk[0], dv[0]
    return BackwardResult(dq, dk, dv, prep.counters(variant, slots))


def run_attention(slots: Sequence[SlotInputs], scale: float, mask, prep: MaskPrep, variant: Variant,
                  threads: int = 1) -> MultiHeadForward:
    """run_attention (engine.hpp:489-505): all slots share the mask and prep. Slots are stacked
    and run as ONE persistent launch (slot-major work list) instead of sequentially."""
    if len(slots) == 0:
        raise ValueError("need at least one batch/head slot")
    d0 = (tuple(slots[0].q.shape[-1:]), tuple(slots[0].v.shape[-1:]))
    for s in slots:
        if (tuple(s.q.shape[-1:]), tuple(s.v.shape[-1:])) != d0:
            raise ValueError("all slots must share head dimensions")
    if isinstance(slots[0].q, np.ndarray):
        q = np.stack([s.q for s in slots])
        k = np.stack([s.k for s in slots])
        v = np.stack([s.v for s in slots])
    else:
        import torch
        q = torch.stack([s.q for s in slots])
        k = torch.stack([s.k for s in slots])
        v = torch.stack([s.v for s in slots])
    res = blocked_forward(q, k, v, scale, mask, prep, variant, threads)
    per = [ForwardResult(res.out[i], res.row_max[i], res.row_sum[i], prep.counters(variant, 1))
           for i in range(len(slots))]
    return MultiHeadForward(per, res.counters)


def run_attention_multi(prep: MaskPrep, variant: Variant, q: np.ndarray, k: np.ndarray, v: np.ndarray,
                        scale: float, devices: Sequence[int]):
    """Multi-GPU driver (C ABI bbm_run_attention_multi): host bf16 (uint16) [slots][n][d] sharded
    contiguously over ``devices``; metadata replicated peer-to-peer. Returns (out, row_max,
    row_sum, elapsed_ms)."""
    slots, n, d = q.shape
    out = np.empty_like(q)
    rmax = np.empty((slots, n), np.float32)
    rsum = np.empty((slots, n), np.float32)
    devs = (C.c_int * len(devices))(*devices)
    ms = C.c_double(0.0)
    check(lib.bbm_run_attention_multi(prep.handle.h, int(variant), len(devices), devs,
                                      ptr(q, C.c_uint16), ptr(k, C.c_uint16), ptr(v, C.c_uint16),
                                      ptr(out, C.c_uint16), ptr(rmax, C.c_float), ptr(rsum, C.c_float),
                                      slots, d, float(scale), C.byref(ms)))
    return out, rmax, rsum, ms.value


def shard_slots(slots: int, world: int, rank: int):
    """Contiguous slot range of one GPU: [r*S/G, (r+1)*S/G)."""
    return slots * rank // world, slots * (rank + 1) // world


# ----------------------------------------------------------------------------- reorder.hpp


@dataclass
class Permutation:
    """reorder.hpp:53-79: forward maps new -> old, inverse old -> new."""
    forward: np.ndarray
    inverse: np.ndarray

    @staticmethod
    def from_forward(fwd) -> "Permutation":
        fwd = np.asarray(fwd, dtype=np.uint32)
        n = fwd.size
        if n and (fwd.max() >= n or np.unique(fwd).size != n):
            raise ValueError("forward map is not a bijection")
        inv = np.empty(n, np.uint32)
        inv[fwd] = np.arange(n, dtype=np.uint32)
        return Permutation(fwd, inv)

    @staticmethod
    def identity(n: int) -> "Permutation":
        return Permutation.from_forward(np.arange(n, dtype=np.uint32))

    def size(self) -> int:
        return int(self.forward.size)


def rcm_order(mask: Mask) -> Permutation:
    """rcm_order(build_graph(mask)) (reorder.hpp:28-133), host."""
    words = np.ascontiguousarray(mask.words)
    fwd = np.zeros(mask.size(), np.uint32)
    check(lib.bbm_rcm_order(ptr(words, C.c_uint64), mask.size(), ptr(fwd, C.c_uint32)))
    return Permutation.from_forward(fwd)


def bandwidth(mask: Mask) -> int:
    """reorder.hpp:137-153"""
    words = np.ascontiguousarray(mask.words)
    out = C.c_uint64(0)
    check(lib.bbm_bandwidth(ptr(words, C.c_uint64), mask.size(), C.byref(out)))
    return int(out.value)


def permute_mask(mask: Mask, perm: Permutation, device: int = 0) -> Mask:
    """permute_mask (reorder.hpp:156-163) on the GPU (K6)."""
    import torch

    if perm.size() != mask.size():
        raise ValueError("permutation length must match mask size")
    dev = torch.device("cuda", device)
    src = torch.from_numpy(np.ascontiguousarray(mask.words).view(np.int64)).to(dev)
    dst = torch.empty_like(src)
    fwd = torch.from_numpy(perm.forward.astype(np.int32)).to(dev)
    with torch.cuda.device(dev):
        check(lib.bbm_permute_mask_device(C.c_void_p(src.data_ptr()), C.c_void_p(dst.data_ptr()),
                                          C.c_void_p(fwd.data_ptr()), mask.size(),
                                          C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)))
    return Mask(mask.size(), dst.cpu().numpy().view(np.uint64))


def _permute_rows_impl(m, perm: Permutation, inverse: bool):
    import torch

    if perm.size() != m.shape[-2]:
        raise ValueError("permutation length must match row count")
    dev = m.device
    fwd = torch.from_numpy(perm.forward.astype(np.int32)).to(dev)
    src = m.contiguous()
    dst = torch.empty_like(src)
    slots = src.numel() // (src.shape[-2] * src.shape[-1])
    row_bytes = src.shape[-1] * src.element_size()
    with torch.cuda.device(dev):
        check(lib.bbm_permute_rows_device(C.c_void_p(src.data_ptr()), C.c_void_p(dst.data_ptr()),
                                          C.c_void_p(fwd.data_ptr()), slots, src.shape[-2], row_bytes,
                                          1 if inverse else 0,
                                          C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)))
    return dst


def permute_rows(m, perm: Permutation):
    """permute_rows (reorder.hpp:167-176) on the GPU (K5): row a <- row forward[a]."""
    return _permute_rows_impl(m, perm, False)


def unpermute_rows(m, perm: Permutation):
    """unpermute_rows (reorder.hpp:180-189) on the GPU (K5): row forward[a] <- row a."""
    return _permute_rows_impl(m, perm, True)


# ----------------------------------------------------------------------------- generators


def generate(spec: str, n: int = 0) -> Mask:
    """MaskSpec::parse + generate (generators.hpp:233-438), host fixture."""
    n_out = C.c_uint64(0)
    check(lib.bbm_generate(spec.encode(), n, C.byref(n_out), None))
    m = Mask(int(n_out.value))
    check(lib.bbm_generate(spec.encode(), n, C.byref(n_out), ptr(m.words, C.c_uint64)))
    return m


def generate_device(spec: str, n: int = 0, device: int = 0, stream=None):
    """generate() straight into device memory: a CUDA int64 tensor [n][ceil(n/64)] holding the
    reference's packed words (bbm_generate_device; random / band families run on the GPU)."""
    import torch

    n_out = C.c_uint64(0)
    check(lib.bbm_generate_device(spec.encode(), n, C.byref(n_out), None, None))
    m = int(n_out.value)
    dev = torch.device("cuda", device)
    words = torch.empty((m, (m + 63) // 64), dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        s = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
        check(lib.bbm_generate_device(spec.encode(), n, C.byref(n_out), C.c_void_p(words.data_ptr()), C.c_void_p(s)))
    return words


def _join(xs: Iterable[int]) -> str:
    return ";".join(str(int(x)) for x in xs)


def gen_causal(n: int) -> Mask:
    return generate("causal", n)


def gen_all_ones(n: int) -> Mask:
    return generate("all-ones", n)


def gen_medusa(candidates: Sequence[int]) -> Mask:
    return generate(f"medusa[{_join(candidates)}]")


def medusa_size(candidates: Sequence[int]) -> int:
    if not candidates:
        raise ValueError("medusa candidate list must be non-empty")
    total, level = 0, 1
    for s in candidates:
        if s < 1:
            raise ValueError("medusa candidate counts must be positive")
        level *= s
        total += level
    return total


def gen_packed_sequential(lengths: Sequence[int]) -> Mask:
    return generate(f"packed-seq[{_join(lengths)}]")


def gen_packed_input_bidirectional(segments: Sequence[tuple]) -> Mask:
    return generate("packed-bidir[" + ";".join(f"{a}:{b}" for a, b in segments) + "]")


def gen_longformer_windowed(n: int, window: int, causal: bool = False) -> Mask:
    return generate(f"windowed(w={window}" + (";causal=1" if causal else "") + ")", n)


def gen_longformer_dilated(n: int, window: int, dilation: int) -> Mask:
    return generate(f"dilated(w={window};d={dilation})", n)


def gen_longformer_global(n: int, window: int, global_count: int) -> Mask:
    return generate(f"global(w={window};g={global_count})", n)


def gen_random_sparse(n: int, density: float, seed: int, force_diagonal: bool = True) -> Mask:
    return generate(f"random(p={density!r};seed={seed}" + ("" if force_diagonal else ";diag=0") + ")", n)


def relabel(mask: Mask, seed: int) -> Mask:
    """out(label[i], label[j]) = mask(i, j), labels = std::shuffle(iota, mt19937_64(seed))."""
    out = Mask(mask.size())
    words = np.ascontiguousarray(mask.words)
    check(lib.bbm_relabel(ptr(words, C.c_uint64), mask.size(), seed, ptr(out.words, C.c_uint64)))
    return out


# ----------------------------------------------------------------------------- mask_io.hpp

MaskIoError = _lib.MaskIoError


def write_mask(mask: Mask, path: str) -> None:
    """write_mask (mask_io.hpp:134-144): "BBMK", version 1, n (u64 LE), ceil(n/8)-byte rows."""
    check(lib.bbm_write_mask_file(str(path).encode(), ptr(mask.words, C.c_uint64), mask.size()))


def read_mask(path: str) -> Mask:
    """read_mask (mask_io.hpp:146-162); raises MaskIoError with the reference's kinds."""
    n = C.c_uint64(0)
    check(lib.bbm_read_mask_file(str(path).encode(), C.byref(n), None))
    m = Mask(int(n.value))
    check(lib.bbm_read_mask_file(str(path).encode(), C.byref(n), ptr(m.words, C.c_uint64)))
    return m


@dataclass
class OccupancyFile:
    """mask_io.hpp:164-168."""
    n_tokens: int
    spec: BlockSpec
    occupancy: BlockOccupancy


def write_occupancy(occ: BlockOccupancy, n_tokens: int, spec: BlockSpec, path: str) -> None:
    """write_occupancy (mask_io.hpp:170-181): the "BBLK" sidecar."""
    vals = np.ascontiguousarray(occ.values, dtype=np.uint8)
    check(lib.bbm_write_occupancy_file(str(path).encode(), ptr(vals, C.c_uint8), n_tokens, spec.block_i,
                                       spec.block_j))


def read_occupancy(path: str) -> OccupancyFile:
    """read_occupancy (mask_io.hpp:183-207)."""
    n, bi, bj = C.c_uint64(0), C.c_uint64(0), C.c_uint64(0)
    check(lib.bbm_read_occupancy_file(str(path).encode(), C.byref(n), C.byref(bi), C.byref(bj), None))
    rows, cols = -(-n.value // bi.value), -(-n.value // bj.value)
    occ = np.zeros((rows, cols), np.uint8)
    check(lib.bbm_read_occupancy_file(str(path).encode(), C.byref(n), C.byref(bi), C.byref(bj),
                                      ptr(occ, C.c_uint8)))
    return OccupancyFile(int(n.value), BlockSpec(int(bi.value), int(bj.value)), BlockOccupancy(occ))


def preprocess_mask_file(path: str, spec: BlockSpec = BlockSpec(), device: int = 0) -> MaskPrep:
    """read_mask + preprocess_mask with the file's byte rows unpacked on the device."""
    spec.validate()
    h = C.c_void_p()
    check(lib.bbm_preprocess_mask_file(str(path).encode(), spec.block_i, spec.block_j, device, C.byref(h)))
    return _prep_from_handle(h)
