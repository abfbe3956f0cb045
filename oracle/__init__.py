"""CPU oracle for the Binary Block Masking hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package, and only as the checker or the timed CPU baseline — never as the product
path. Two layers:

* ``liboracle.so``   the plain-C restatement (bbm_oracle.c), each function citing the reference
                     file:line it follows;
* ``_ref/libbbm_ref.so``  the UNMODIFIED reference headers compiled in place (ref_shim.cpp),
                     present when the build ran where /root/reference exists (it travels to the
                     GPU box as a prebuilt file). Used to pin the restatement and as the CPU
                     baseline (``cpu_baseline.kind = "reference"``).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_PATH = os.path.join(_HERE, "liboracle.so")
REF_PATH = os.path.join(_HERE, "_ref", "libbbm_ref.so")

_orc = None
_ref = None

u8p, u32p, u64p = C.POINTER(C.c_uint8), C.POINTER(C.c_uint32), C.POINTER(C.c_uint64)
f32p, f64p, vp = C.POINTER(C.c_float), C.POINTER(C.c_double), C.c_void_p


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


class Counters(C.Structure):
    _fields_ = [("blocks_visited", C.c_uint64), ("blocks_processed", C.c_uint64),
                ("mask_block_reads", C.c_uint64), ("skipped_by_binblk", C.c_uint64),
                ("skipped_mask_reads_by_run", C.c_uint64)]

    def as_tuple(self):
        return (self.blocks_visited, self.blocks_processed, self.mask_block_reads,
                self.skipped_by_binblk, self.skipped_mask_reads_by_run)


class Stats(C.Structure):
    _fields_ = [("blocks_total", C.c_uint64), ("blocks_nonzero", C.c_uint64),
                ("blocks_full", C.c_uint64), ("block_density", C.c_double),
                ("element_density", C.c_double)]


def orc():
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_PATH):
            raise ImportError(f"{ORACLE_PATH} missing: run `make -C oracle`")
        L = C.CDLL(ORACLE_PATH)
        L.orc_make_problem.argtypes = [C.c_uint64] * 4 + [f64p] * 4
        L.orc_block_sums.argtypes = [u64p, C.c_uint64, C.c_uint64, C.c_uint64, u32p]
        L.orc_block_occupancy.argtypes = [u32p, C.c_uint64, C.c_uint64, u8p]
        L.orc_dense_runs.argtypes = [u32p, C.c_uint64, C.c_uint64, C.c_uint64, u32p, u32p]
        L.orc_block_stats.argtypes = [u32p, C.c_uint64, C.c_uint64, C.c_uint64, C.POINTER(Stats)]
        L.orc_counters.argtypes = [u32p, u32p, u32p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int,
                                   C.POINTER(Counters)]
        L.orc_naive_forward.argtypes = [f64p, f64p, f64p, C.c_uint64, C.c_uint64, C.c_uint64,
                                        C.c_double, u64p, f64p, f64p, f64p, C.c_int]
        L.orc_dense_forward.argtypes = [f64p, f64p, f64p, C.c_uint64, C.c_uint64, C.c_uint64,
                                        C.c_double, f64p, f64p, f64p, C.c_int]
        L.orc_naive_backward.argtypes = [f64p, f64p, f64p, f64p, C.c_uint64, C.c_uint64, C.c_double,
                                         u64p, f64p, f64p, f64p, C.c_int]
        L.orc_naive_rows.argtypes = [f64p, f64p, f64p, f64p, C.c_uint64, C.c_uint64, C.c_double, u64p,
                                     u64p, C.c_uint64, f64p, f64p, f64p, f64p]
        L.orc_rcm_order.argtypes = [u64p, C.c_uint64, u32p]
        L.orc_bandwidth.argtypes = [u64p, C.c_uint64]
        L.orc_bandwidth.restype = C.c_uint64
        L.orc_permute_mask.argtypes = [u64p, C.c_uint64, u32p, u64p]
        L.orc_permute_rows.argtypes = [vp, vp, C.c_uint64, C.c_uint64, u32p, C.c_int]
        _orc = L
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref():
    global _ref
    if _ref is None:
        if not ref_available():
            raise ImportError(f"{REF_PATH} missing (built only where /root/reference exists)")
        L = C.CDLL(REF_PATH)
        L.ref_last_error.restype = C.c_char_p
        L.ref_generate.argtypes = [C.c_char_p, C.c_uint64, u64p, u64p]
        L.ref_preprocess.argtypes = [u64p, C.c_uint64, C.c_uint64, C.c_uint64, u32p, u8p, u32p, u32p,
                                     u64p, f64p]
        L.ref_blocked_forward.argtypes = [C.c_int, vp, vp, vp, C.c_uint64, C.c_uint64, C.c_uint64,
                                          C.c_double, u64p, C.c_uint64, C.c_uint64, C.c_int, C.c_uint,
                                          vp, f64p, f64p, u64p]
        L.ref_engine_create.argtypes = [u64p, C.c_uint64, C.c_uint64, C.c_uint64, f32p, f32p, f32p,
                                        C.c_uint64, C.c_uint64]
        L.ref_engine_create.restype = vp
        L.ref_engine_forward.argtypes = [vp, C.c_int, C.c_uint, C.c_double]
        L.ref_engine_forward.restype = C.c_double
        L.ref_engine_preprocess_ms.argtypes = [vp, C.c_int]
        L.ref_engine_preprocess_ms.restype = C.c_double
        L.ref_engine_destroy.argtypes = [vp]
        L.ref_naive_forward.argtypes = [f64p, f64p, f64p, C.c_uint64, C.c_uint64, C.c_uint64,
                                        C.c_double, u64p, f64p, f64p, f64p]
        L.ref_naive_backward.argtypes = [f64p, f64p, f64p, C.c_uint64, C.c_uint64, C.c_double, u64p,
                                         f64p, f64p, f64p, f64p]
        L.ref_rcm.argtypes = [u64p, C.c_uint64, u32p, u64p, u64p]
        L.ref_permute_mask.argtypes = [u64p, C.c_uint64, u32p, u64p]
        L.ref_relabel.argtypes = [u64p, C.c_uint64, C.c_uint64, u64p]
        L.ref_make_problem_f32.argtypes = [C.c_uint64] * 4 + [f32p] * 4
        _ref = L
    return _ref


def _check_ref(rc):
    if rc != 0:
        raise ValueError(ref().ref_last_error().decode())


# ------------------------------------------------------------------ oracle (C restatement)

def make_problem(seed: int, slots: int, n: int, d: int):
    """(q, k, v, d_out) float64 [slots][n][d], the make_problem stream (bench.hpp:320-337)."""
    arrs = [np.empty((slots, n, d), np.float64) for _ in range(4)]
    orc().orc_make_problem(seed, slots, n, d, *[_p(a, C.c_double) for a in arrs])
    return tuple(arrs)


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bf16, returned as float64 (what the GPU sees)."""
    f = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (f >> 16) & 1
    r = ((f + 0x7FFF + lsb) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).astype(np.float64)


def block_sums(words: np.ndarray, n: int, bi: int, bj: int) -> np.ndarray:
    rows, cols = -(-n // bi), -(-n // bj)
    out = np.zeros((rows, cols), np.uint32)
    w = np.ascontiguousarray(words, dtype=np.uint64)
    orc().orc_block_sums(_p(w, C.c_uint64), n, bi, bj, _p(out, C.c_uint32))
    return out


def preprocess(words: np.ndarray, n: int, bi: int, bj: int):
    """(sums, occ, offset, total_ones, stats dict) per mask.hpp:184-247."""
    sums = block_sums(words, n, bi, bj)
    rows, cols = sums.shape
    occ = np.zeros((rows, cols), np.uint8)
    off = np.zeros(rows, np.uint32)
    tot = np.zeros(rows, np.uint32)
    st = Stats()
    L = orc()
    L.orc_block_occupancy(_p(sums, C.c_uint32), rows, cols, _p(occ, C.c_uint8))
    L.orc_dense_runs(_p(sums, C.c_uint32), n, bi, bj, _p(off, C.c_uint32), _p(tot, C.c_uint32))
    L.orc_block_stats(_p(sums, C.c_uint32), n, bi, bj, C.byref(st))
    stats = dict(blocks_total=st.blocks_total, blocks_nonzero=st.blocks_nonzero,
                 blocks_full=st.blocks_full, block_density=st.block_density,
                 element_density=st.element_density)
    return sums, occ, off, tot, stats


def counters(words, n, bi, bj, variant: int):
    sums, _, off, tot, _ = preprocess(words, n, bi, bj)
    c = Counters()
    orc().orc_counters(_p(sums, C.c_uint32), _p(off, C.c_uint32), _p(tot, C.c_uint32), n, bi, bj,
                       variant, C.byref(c))
    return c.as_tuple()


def naive_forward(q, k, v, scale: float, words, n: int, threads: int = 8):
    """reference.hpp:42-81 in double; q,k,v [n][d] float64. words=None -> every key visible
    (the dense variant)."""
    q, k, v = (np.ascontiguousarray(a, dtype=np.float64) for a in (q, k, v))
    d, dv = q.shape[1], v.shape[1]
    out = np.zeros((n, dv), np.float64)
    rmax = np.zeros(n, np.float64)
    rsum = np.zeros(n, np.float64)
    L = orc()
    if words is None:
        L.orc_dense_forward(_p(q, C.c_double), _p(k, C.c_double), _p(v, C.c_double), n, d, dv, scale,
                            _p(out, C.c_double), _p(rmax, C.c_double), _p(rsum, C.c_double), threads)
    else:
        w = np.ascontiguousarray(words, dtype=np.uint64)
        L.orc_naive_forward(_p(q, C.c_double), _p(k, C.c_double), _p(v, C.c_double), n, d, dv, scale,
                            _p(w, C.c_uint64), _p(out, C.c_double), _p(rmax, C.c_double),
                            _p(rsum, C.c_double), threads)
    return out, rmax, rsum


def naive_backward(q, k, v, d_out, scale: float, words, n: int, threads: int = 8):
    """reference.hpp:84-139 in double: (dq, dk, dv) of L = sum(out * d_out). words=None -> every
    key visible (the dense variant)."""
    q, k, v, g = (np.ascontiguousarray(a, dtype=np.float64) for a in (q, k, v, d_out))
    d = q.shape[1]
    dq, dk, dv = (np.zeros((n, d), np.float64) for _ in range(3))
    w = None if words is None else np.ascontiguousarray(words, dtype=np.uint64)
    orc().orc_naive_backward(_p(q, C.c_double), _p(k, C.c_double), _p(v, C.c_double), _p(g, C.c_double),
                             n, d, scale, None if w is None else _p(w, C.c_uint64), _p(dq, C.c_double),
                             _p(dk, C.c_double), _p(dv, C.c_double), threads)
    return dq, dk, dv


def naive_rows(q, k, v, scale: float, words, n: int, rows, d_out=None):
    """Forward (out, row_max, row_sum) and, with d_out, dq of the listed query rows only
    (reference.hpp:42-139 restated per row); q, k, v, d_out [n][d]. words=None: dense."""
    q, k, v = (np.ascontiguousarray(a, dtype=np.float64) for a in (q, k, v))
    g = None if d_out is None else np.ascontiguousarray(d_out, dtype=np.float64)
    r = np.ascontiguousarray(rows, dtype=np.uint64)
    d = q.shape[1]
    out = np.zeros((r.size, d), np.float64)
    rmax = np.zeros(r.size, np.float64)
    rsum = np.zeros(r.size, np.float64)
    dq = None if g is None else np.zeros((r.size, d), np.float64)
    w = None if words is None else np.ascontiguousarray(words, dtype=np.uint64)
    orc().orc_naive_rows(_p(q, C.c_double), _p(k, C.c_double), _p(v, C.c_double),
                         None if g is None else _p(g, C.c_double), n, d, scale,
                         None if w is None else _p(w, C.c_uint64), _p(r, C.c_uint64), r.size,
                         _p(out, C.c_double), _p(rmax, C.c_double), _p(rsum, C.c_double),
                         None if dq is None else _p(dq, C.c_double))
    return out, rmax, rsum, dq


def ref_naive_backward(q, k, v, d_out, scale: float, words, n: int):
    """The reference's own naive_backward (oracle/_ref), to pin the restatement."""
    q, k, v, g = (np.ascontiguousarray(a, dtype=np.float64) for a in (q, k, v, d_out))
    d = q.shape[1]
    dq, dk, dv = (np.zeros((n, d), np.float64) for _ in range(3))
    w = np.ascontiguousarray(words, dtype=np.uint64)
    _check_ref(ref().ref_naive_backward(_p(q, C.c_double), _p(k, C.c_double), _p(v, C.c_double), n, d, scale,
                                        _p(w, C.c_uint64), _p(g, C.c_double), _p(dq, C.c_double),
                                        _p(dk, C.c_double), _p(dv, C.c_double)))
    return dq, dk, dv


def rcm_order(words, n: int) -> np.ndarray:
    fwd = np.zeros(n, np.uint32)
    w = np.ascontiguousarray(words, dtype=np.uint64)
    orc().orc_rcm_order(_p(w, C.c_uint64), n, _p(fwd, C.c_uint32))
    return fwd


def bandwidth(words, n: int) -> int:
    w = np.ascontiguousarray(words, dtype=np.uint64)
    return int(orc().orc_bandwidth(_p(w, C.c_uint64), n))


def permute_mask(words, n: int, fwd) -> np.ndarray:
    w = np.ascontiguousarray(words, dtype=np.uint64)
    f = np.ascontiguousarray(fwd, dtype=np.uint32)
    out = np.zeros_like(w)
    orc().orc_permute_mask(_p(w, C.c_uint64), n, _p(f, C.c_uint32), _p(out, C.c_uint64))
    return out


# ------------------------------------------------------------------ real reference (_ref)

def ref_generate(spec: str, n: int = 0) -> np.ndarray:
    L = ref()
    n_out = C.c_uint64(0)
    _check_ref(L.ref_generate(spec.encode(), n, C.byref(n_out), None))
    m = int(n_out.value)
    words = np.zeros((m, (m + 63) // 64), np.uint64)
    _check_ref(L.ref_generate(spec.encode(), n, C.byref(n_out), _p(words, C.c_uint64)))
    return words


def ref_preprocess(words, n, bi, bj):
    rows, cols = -(-n // bi), -(-n // bj)
    sums = np.zeros((rows, cols), np.uint32)
    occ = np.zeros((rows, cols), np.uint8)
    off = np.zeros(rows, np.uint32)
    tot = np.zeros(rows, np.uint32)
    su = np.zeros(3, np.uint64)
    sf = np.zeros(2, np.float64)
    w = np.ascontiguousarray(words, dtype=np.uint64)
    _check_ref(ref().ref_preprocess(_p(w, C.c_uint64), n, bi, bj, _p(sums, C.c_uint32), _p(occ, C.c_uint8),
                                    _p(off, C.c_uint32), _p(tot, C.c_uint32), _p(su, C.c_uint64),
                                    _p(sf, C.c_double)))
    stats = dict(blocks_total=int(su[0]), blocks_nonzero=int(su[1]), blocks_full=int(su[2]),
                 block_density=float(sf[0]), element_density=float(sf[1]))
    return sums, occ, off, tot, stats


def ref_blocked_forward(q, k, v, scale, words, n, bi, bj, variant, threads=8, dtype=np.float32):
    """blocked_forward<T> over stacked slots [slots][n][d]; returns out, row_max, row_sum,
    counters (5-tuple)."""
    q, k, v = (np.ascontiguousarray(a, dtype=dtype) for a in (q, k, v))
    slots, _, d = q.shape
    out = np.zeros_like(q)
    rmax = np.zeros((slots, n), np.float64)
    rsum = np.zeros((slots, n), np.float64)
    cnt = np.zeros(5, np.uint64)
    w = np.ascontiguousarray(words, dtype=np.uint64)
    _check_ref(ref().ref_blocked_forward(1 if dtype == np.float64 else 0, q.ctypes.data, k.ctypes.data,
                                         v.ctypes.data, slots, n, d, scale, _p(w, C.c_uint64), bi, bj,
                                         variant, threads, out.ctypes.data, _p(rmax, C.c_double),
                                         _p(rsum, C.c_double), _p(cnt, C.c_uint64)))
    return out, rmax, rsum, tuple(int(x) for x in cnt)


def ref_rcm(words, n):
    fwd = np.zeros(n, np.uint32)
    bw0, bw1 = C.c_uint64(0), C.c_uint64(0)
    w = np.ascontiguousarray(words, dtype=np.uint64)
    _check_ref(ref().ref_rcm(_p(w, C.c_uint64), n, _p(fwd, C.c_uint32), C.byref(bw0), C.byref(bw1)))
    return fwd, int(bw0.value), int(bw1.value)


def ref_make_problem_f32(seed, slots, n, d):
    arrs = [np.empty((slots, n, d), np.float32) for _ in range(4)]
    ref().ref_make_problem_f32(seed, slots, n, d, *[_p(a, C.c_float) for a in arrs])
    return tuple(arrs)


def ref_permute_mask(words, n, fwd):
    """The reference's permute_mask (reorder.hpp:156-163): out(a, b) = mask(fwd[a], fwd[b])."""
    w = np.ascontiguousarray(words, dtype=np.uint64)
    f = np.ascontiguousarray(fwd, dtype=np.uint32)
    out = np.zeros_like(w)
    _check_ref(ref().ref_permute_mask(_p(w, C.c_uint64), n, _p(f, C.c_uint32), _p(out, C.c_uint64)))
    return out


def ref_relabel(words, n, seed):
    """Config 5's shuffle relabelling through the reference's permute_mask (ref_shim.cpp)."""
    w = np.ascontiguousarray(words, dtype=np.uint64)
    out = np.zeros_like(w)
    _check_ref(ref().ref_relabel(_p(w, C.c_uint64), n, seed, _p(out, C.c_uint64)))
    return out
