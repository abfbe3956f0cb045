"""B200-native Binary Block Masking (arXiv 2409.15097).

A drop-in for the reference's hot path (mask preprocessing + block-sparse masked attention
forward, namespace blockmask in /root/reference/proj/include): host code mirrors the reference
API (``blockmask``), every compute call goes through the C ABI of ``libbbm.so`` to hand-written
sm_100a kernels. Importing fails loudly if the library was not built: there is no CPU fallback.
"""
from . import _lib  # noqa: F401  (raises ImportError when libbbm.so is missing)
from .blockmask import *  # noqa: F401,F403
from .blockmask import (BackwardResult, attn_bwd_device, blocked_backward)  # noqa: F401
from .blockmask import (MaskIoError, OccupancyFile, preprocess_mask_file, read_mask, read_occupancy,  # noqa: F401
                        write_mask, write_occupancy)
from .blockmask import (BlockOccupancy, BlockSpec, BlockStats, BlockSums, DenseRuns, EngineCounters,
                        ForwardResult, Mask, MaskPrep, MultiHeadForward, Permutation, SlotInputs,
                        Variant, attn_fwd_device, bandwidth, block_stats, block_sums,
                        blocked_forward, build_block_occupancy, build_dense_runs, generate,
                        parse_variant, permute_mask, permute_rows, preprocess_mask, rcm_order,
                        generate_device, import_prep_ipc, relabel, run_attention, run_attention_multi, shard_slots, to_string,
                        unpermute_rows)

LIB_PATH = _lib.LIB_PATH
