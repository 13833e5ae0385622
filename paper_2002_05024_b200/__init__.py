"""B200-native (sm_100a) window-based off-diagonal update path of StarNEig
(arXiv 2002.05024): Schur-form eigenvalue reordering and multishift QR with
aggressive early deflation (Schur reduction) behind the reference's ``taskeig`` API.

The compute path is the in-tree CUDA library ``_lib/libtaskeig_b200.so``
(C ABI: ``include/taskeig_b200.h``); this package is the host-side mirror of
the reference interface.  There is no CPU fallback.
"""
from ._native import (TaskeigError, build, host_transfer_bytes, lib, memory_retention, release_memory,  # noqa: F401
                      set_memory_retention,
                      trace_enable, trace_json)
from .reorder import (  # noqa: F401
    Block, GReorderResult, PlanWindow, ReorderOptions, ReorderResult, Selection, WindowReorderOutcome,
    gen_pair_t, greorder_schur,
    apply_window_updates, colmajor_empty, gen_hessenberg, gen_schur_input, identity,
    known_spectrum_seed, plan_reorder, reorder_schur, scan_blocks, scan_blocks_device, select_by_name,
    select_eigenvalues, select_fraction, window_reorder)
from .eigvec import backtransform  # noqa: F401
from .hessenberg import HessenbergOptions, HessenbergResult, hessenberg_reduce  # noqa: F401
from . import io  # noqa: F401  (matrix files: T.io.read_matrix_file / write_matrix_file)
from .schur import (  # noqa: F401
    AedResult, BulgeChain, DeflationCondition, SchurDecomposition, SchurOptions, aed_step, chase_bulges,
    deflation_check, introduce_bulges, schur_reduce, small_schur)

__all__ = [n for n in dir() if not n.startswith("_")]
