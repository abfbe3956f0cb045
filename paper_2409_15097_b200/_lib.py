"""ctypes binding of libbbm.so (include/bbm_capi.h).

The library is built in-tree (``__graft_entry__.build()`` / ``make -C paper_2409_15097_b200/csrc``).
There is no fallback: if the shared object is missing, importing the package raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libbbm.so")
# A/B timing experiments (tools/ablate.sh) may point at another in-tree build of the same library
LIB_PATH = os.environ.get("BBM_LIB", LIB_PATH)

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"libbbm.so not found at {LIB_PATH}: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        " (there is no CPU fallback for the B200 engine)")

lib = C.CDLL(LIB_PATH)

u8p = C.POINTER(C.c_uint8)
u16p = C.POINTER(C.c_uint16)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
f32p = C.POINTER(C.c_float)
f64p = C.POINTER(C.c_double)
vp = C.c_void_p

BBM_OK, BBM_ERR_INVALID, BBM_ERR_CUDA, BBM_ERR_UNSUPPORTED, BBM_ERR_INTERNAL = range(5)
# MaskIoError kinds (mask_io.hpp:24-42)
IO_KINDS = {10: "io_failure", 11: "bad_magic", 12: "bad_version", 13: "dimension_overflow",
            14: "truncated", 15: "trailing_data"}


class BlockStatsC(C.Structure):
    _fields_ = [("blocks_total", C.c_uint64), ("blocks_nonzero", C.c_uint64),
                ("blocks_full", C.c_uint64), ("block_density", C.c_double),
                ("element_density", C.c_double)]


class CountersC(C.Structure):
    _fields_ = [("blocks_visited", C.c_uint64), ("blocks_processed", C.c_uint64),
                ("mask_block_reads", C.c_uint64), ("skipped_by_binblk", C.c_uint64),
                ("skipped_mask_reads_by_run", C.c_uint64)]


class PrepInfoC(C.Structure):
    _fields_ = [("n", C.c_uint64), ("block_i", C.c_uint64), ("block_j", C.c_uint64),
                ("rows", C.c_uint64), ("cols", C.c_uint64), ("ktile", C.c_uint32),
                ("krows", C.c_uint32), ("kcols", C.c_uint32), ("knnz", C.c_uint64),
                ("kfull", C.c_uint64), ("device", C.c_int)]


# name -> (restype, argtypes); every symbol declared in include/bbm_capi.h
SIGNATURES = {
    "bbm_abi_version": (C.c_int, []),
    "bbm_last_error": (C.c_char_p, []),
    "bbm_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "bbm_preprocess_packed_host": (C.c_int, [u64p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, C.POINTER(vp)]),
    "bbm_preprocess_packed_device": (C.c_int, [vp, C.c_uint64, C.c_uint64, C.c_uint64, vp, C.POINTER(vp)]),
    "bbm_preprocess_bool_device": (C.c_int, [vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, vp, C.POINTER(vp)]),
    "bbm_prep_update_bool_device": (C.c_int, [vp, vp, C.c_uint64, vp]),
    "bbm_prep_update_packed_device": (C.c_int, [vp, vp, vp]),
    "bbm_prep_destroy": (C.c_int, [vp]),
    "bbm_prep_get_info": (C.c_int, [vp, C.POINTER(PrepInfoC)]),
    "bbm_prep_get_sums": (C.c_int, [vp, u32p]),
    "bbm_prep_get_occupancy": (C.c_int, [vp, u8p]),
    "bbm_prep_get_runs": (C.c_int, [vp, u32p, u32p]),
    "bbm_prep_get_stats": (C.c_int, [vp, C.POINTER(BlockStatsC)]),
    "bbm_prep_get_tile_halves": (C.c_int, [vp, vp]),
    "bbm_prep_get_kernel_lists": (C.c_int, [vp, u32p, u32p, u32p]),
    "bbm_prep_counters": (C.c_int, [vp, C.c_int, C.c_uint64, C.POINTER(CountersC)]),
    "bbm_prep_replicate": (C.c_int, [vp, C.c_int, vp, C.POINTER(vp)]),
    "bbm_prep_export_ipc": (C.c_int, [vp, vp, C.POINTER(C.c_size_t)]),
    "bbm_prep_import_ipc": (C.c_int, [vp, C.c_size_t, C.c_int, vp, C.POINTER(vp)]),
    "bbm_sums_metadata": (C.c_int, [u32p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, u8p, u32p, u32p, C.POINTER(BlockStatsC)]),
    "bbm_attn_bwd": (C.c_int, [vp, C.c_int, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, C.c_uint64, C.c_uint32, C.c_double, vp]),
    "bbm_attn_bwd_host_f32": (C.c_int, [vp, C.c_int, f32p, f32p, f32p, f32p, f64p, f64p, f32p, f32p, f32p, f32p, C.c_uint64, C.c_uint32, C.c_double]),
    "bbm_attn_bwd_host_f32_dims": (C.c_int, [vp, C.c_int, f32p, f32p, f32p, f32p, f64p, f64p, f32p, f32p, f32p, f32p,
                                             C.c_uint64, C.c_uint32, C.c_uint32, C.c_double]),
    "bbm_permute_rows_host": (C.c_int, [vp, vp, u32p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, C.c_int]),
    "bbm_permute_mask_host": (C.c_int, [u64p, u64p, u32p, C.c_uint64, C.c_int]),
    "bbm_graph_csr": (C.c_int, [u64p, C.c_uint64, u64p, u32p]),
    "bbm_attn_fwd": (C.c_int, [vp, C.c_int, vp, vp, vp, vp, vp, vp, C.c_uint64, C.c_uint32, C.c_double, vp]),
    "bbm_attn_fwd_gather": (C.c_int, [vp, C.c_int, vp, vp, vp, vp, vp, vp, vp, C.c_uint64, C.c_uint32, C.c_double, vp]),
    "bbm_attn_fwd_gather_ex": (C.c_int, [vp, C.c_int, vp, vp, vp, vp, vp, vp, vp, C.c_uint64, C.c_uint32, C.c_double, vp,
                                         C.c_int]),
    "bbm_attn_fwd_host_bf16": (C.c_int, [vp, C.c_int, u16p, u16p, u16p, u16p, f32p, f32p, C.c_uint64, C.c_uint32, C.c_double]),
    "bbm_attn_fwd_rcm_host_bf16": (C.c_int, [vp, C.c_int, u32p, u16p, u16p, u16p, u16p, f32p, f32p, C.c_uint64, C.c_uint32, C.c_double]),
    "bbm_attn_fwd_host_f32": (C.c_int, [vp, C.c_int, f32p, f32p, f32p, f32p, f64p, f64p, C.c_uint64, C.c_uint32, C.c_double]),
    "bbm_run_attention_host_f32": (C.c_int, [vp, C.c_int, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), C.POINTER(vp),
                                             C.POINTER(vp), C.POINTER(vp), C.c_uint64, C.c_uint32, C.c_double]),
    "bbm_run_attention_host_f32_dims": (C.c_int, [vp, C.c_int, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp),
                                                  C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), C.c_uint64,
                                                  C.c_uint32, C.c_uint32, C.c_double]),
    "bbm_run_attention_multi": (C.c_int, [vp, C.c_int, C.c_int, C.POINTER(C.c_int), u16p, u16p, u16p, u16p, f32p, f32p, C.c_uint64, C.c_uint32, C.c_double, f64p]),
    "bbm_set_trace": (C.c_int, [vp, C.c_uint32]),
    "bbm_set_fwd_kernel": (C.c_int, [C.c_int]),
    "bbm_fwd_build_counts": (C.c_int, [C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "bbm_rcm_order": (C.c_int, [u64p, C.c_uint64, u32p]),
    "bbm_bandwidth": (C.c_int, [u64p, C.c_uint64, u64p]),
    "bbm_permute_rows_device": (C.c_int, [vp, vp, vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, vp]),
    "bbm_permute_mask_device": (C.c_int, [vp, vp, vp, C.c_uint64, vp]),
    "bbm_generate": (C.c_int, [C.c_char_p, C.c_uint64, u64p, u64p]),
    "bbm_generate_device": (C.c_int, [C.c_char_p, C.c_uint64, u64p, vp, vp]),
    "bbm_relabel": (C.c_int, [u64p, C.c_uint64, C.c_uint64, u64p]),
    "bbm_write_mask_file": (C.c_int, [C.c_char_p, u64p, C.c_uint64]),
    "bbm_read_mask_file": (C.c_int, [C.c_char_p, u64p, u64p]),
    "bbm_write_occupancy_file": (C.c_int, [C.c_char_p, u8p, C.c_uint64, C.c_uint64, C.c_uint64]),
    "bbm_read_occupancy_file": (C.c_int, [C.c_char_p, u64p, u64p, u64p, u8p]),
    "bbm_preprocess_mask_file": (C.c_int, [C.c_char_p, C.c_uint64, C.c_uint64, C.c_int, C.POINTER(vp)]),
    "bbm_make_problem": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, f32p, f32p, f32p, f32p]),
}

for _name, (_res, _args) in SIGNATURES.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


class BbmError(RuntimeError):
    """CUDA / internal failure inside libbbm."""


class MaskIoError(RuntimeError):
    """mask_io.hpp:24-42: a mask / occupancy file problem; ``kind`` names which."""

    def __init__(self, kind: str, msg: str):
        super().__init__(msg)
        self.kind = kind


def check(status: int) -> None:
    """Map a bbm_status to the reference's error convention (matrix.hpp:47-49)."""
    if status == BBM_OK:
        return
    msg = lib.bbm_last_error().decode(errors="replace")
    if status in IO_KINDS:
        raise MaskIoError(IO_KINDS[status], msg)
    if status in (BBM_ERR_INVALID, BBM_ERR_UNSUPPORTED):
        raise ValueError(msg)  # the Python spelling of std::invalid_argument
    raise BbmError(msg)


def ptr(arr, ctype):
    """numpy array -> typed ctypes pointer (arr must stay alive)."""
    return arr.ctypes.data_as(C.POINTER(ctype))
