"""ctypes binding of ``libkifmm_b200.so`` (the C-ABI in include/kifmm_b200.h).

There is no fallback: if the shared library is missing or no CUDA device is
visible, every device entry point raises.  Build the library with
``python -c "import __graft_entry__ as g; g.build()"`` (or ``make -C
paper_2408_07436_b200``).
"""

from __future__ import annotations

import ctypes
import os

LIB_NAME = "libkifmm_b200.so"
LIB_PATH = os.environ.get("KIFMM_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), LIB_NAME)     # KIFMM_LIB: variant builds (tools)

_P = ctypes.c_void_p
_I = ctypes.c_int64
_F = ctypes.c_float
_D = ctypes.c_double
_C = ctypes.c_int

# name -> argument types (all return int status)
SIGNATURES = {
    "kifmm_laplace_potentials_f32": [_P, _P, _P, _I, _P, _P, _P, _I, _P, _I, _P, _P],
    "kifmm_laplace_potentials_f64": [_P, _P, _P, _I, _P, _P, _P, _I, _P, _I, _P, _P],
    "kifmm_tree_temp_bytes": [_C, _I, _C, _P],
    "kifmm_tree_encode": [_P, _I, _D, _D, _D, _D, _I, _P, _P, _P],
    "kifmm_tree_sort": [_P, _I, _C, _P, _P, _P, _I, _P],
    "kifmm_tree_rle": [_P, _I, _P, _P, _P, _P, _I, _P],
    "kifmm_tree_parents": [_P, _I, _P, _P, _P, _P, _I, _P],
    "kifmm_lookup_codes": [_P, _I, _P, _I, _P, _P],
    "kifmm_near_field_rows": [_P, _I, _I, _P, _I, _P, _P],
    "kifmm_blas_src_table": [_P, _P, _I, _I, _P, _P, _P, _I, _P, _P],
    "kifmm_laplace_gradients_f32": [_P, _P, _P, _I, _P, _P, _P, _I, _P, _I, _P, _P, _P],
    "kifmm_laplace_gradients_f64": [_P, _P, _P, _I, _P, _P, _P, _I, _P, _I, _P, _P, _P],
    "kifmm_laplace_matrix_f32": [_P, _P, _P, _I, _P, _P, _P, _I, _P, _P],
    "kifmm_laplace_matrix_f64": [_P, _P, _P, _I, _P, _P, _P, _I, _P, _P],
    "kifmm_p2p_blocked_f32": [_P, _P, _P, _I, _P, _P, _P, _P, _P, _I, _P, _I, _P, _P],
    "kifmm_p2p_blocked_f64": [_P, _P, _P, _I, _P, _P, _P, _P, _P, _I, _P, _I, _P, _P],
    "kifmm_hadamard_m2l_c64": [_P, _P, _P, _P, _I, _I, _I, _I, _P],
    "kifmm_hadamard_m2l_c128": [_P, _P, _P, _P, _I, _I, _I, _I, _P],
    "kifmm_hadamard_tiled_c64": [_P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _C, _P, _P],
    "kifmm_hadamard_tiled_c128": [_P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _C, _P, _P],
    "kifmm_gemm_f32": [_I, _I, _I, _F, _P, _I, _C, _I, _P, _I, _P, _P, _I, _P, _C, _P],
    "kifmm_gemm_f64": [_I, _I, _I, _D, _P, _I, _C, _I, _P, _I, _P, _P, _I, _P, _C, _P],
    "kifmm_p2m_check_f32": [_P, _P, _P, _P, _I, _P, _P, _I, _P, _P, _I, _P, _P],
    "kifmm_p2m_check_f64": [_P, _P, _P, _P, _I, _P, _P, _I, _P, _P, _I, _P, _P],
    "kifmm_stack_children_f32": [_P, _P, _I, _I, _I, _P, _P],
    "kifmm_stack_children_f64": [_P, _P, _I, _I, _I, _P, _P],
    "kifmm_m2l_sweep_f32": [_P, _P, _I, _I, _P, _P, _P, _P, _I, _I, _I, _P, _P],
    "kifmm_m2l_sweep_f64": [_P, _P, _I, _I, _P, _P, _P, _P, _I, _I, _I, _P, _P],
    "kifmm_m2l_sweep_sparse_f64": [_P, _P, _I, _I, _P, _P, _P, _P, _I, _I, _I, _P, _P, _P, _P,
                                   _P],
    "kifmm_fft_forward_f32": [_P, _I, _I, _P, _I, _P, _I, _P, _P],
    "kifmm_fft_forward_f64": [_P, _I, _I, _P, _I, _P, _I, _P, _P],
    "kifmm_gather_rows_f32": [_P, _P, _I, _I, _P, _P],
    "kifmm_gather_rows_f64": [_P, _P, _I, _I, _P, _P],
    "kifmm_scatter_rows_f32": [_P, _P, _I, _I, _P, _P],
    "kifmm_scatter_rows_f64": [_P, _P, _I, _I, _P, _P],
    "kifmm_m2l_compress_f64": [_P, _I, _I, _P, _P, _P, _P, _P, _P, _I, _I, _I, _P, _P, _I, _P],
    "kifmm_m2l_expand_f64": [_P, _I, _P, _P, _P, _I, _P, _P, _P, _P, _I, _I, _I, _P, _P, _P, _P,
                             _P],
    "kifmm_rowchain_f32": [_I, _P, _I, _I, _I, _I, _P, _P, _P, _I, _I, _I, _I, _P, _P, _P, _F, _F, _F,
                           _P, _P, _P, _I, _I, _I, _P, _P, _P, _I, _I, _I, _P],
    "kifmm_move_rows_f32": [_P, _P, _P, _I, _I, _P, _P],
    "kifmm_move_rows_f64": [_P, _P, _P, _I, _I, _P, _P],
    "kifmm_fft_inverse_f32": [_P, _I, _I, _P, _I, _D, _P, _P],
    "kifmm_fft_inverse_f64": [_P, _I, _I, _P, _I, _D, _P, _P],
    "kifmm_leaf_pass_f32": [_P, _P, _P, _P, _P, _I, _P, _P, _I, _P, _P, _I, _P, _P, _P, _P,
                            _I, _P, _C, _P, _P],
    "kifmm_leaf_pass_f64": [_P, _P, _P, _P, _P, _I, _P, _P, _I, _P, _P, _I, _P, _P, _P, _P,
                            _I, _P, _C, _P, _P],
    "kifmm_leaf_pass_grad_f32": [_P, _P, _P, _P, _P, _I, _P, _P, _I, _P, _P, _I, _P, _P, _P,
                                 _P, _I, _P, _C, _P, _P, _P],
    "kifmm_leaf_pass_grad_f64": [_P, _P, _P, _P, _P, _I, _P, _P, _I, _P, _P, _I, _P, _P, _P,
                                 _P, _I, _P, _C, _P, _P, _P],
    "kifmm_pack_sources_f32": [_P, _P, _P, _P, _I, _I, _P, _P],
    "kifmm_pack_sources_f64": [_P, _P, _P, _P, _I, _I, _P, _P],
    "kifmm_l2p_add_f32": [_P, _P, _P, _P, _P, _I, _P, _P, _I, _P, _I, _P, _P, _P, _P],
    "kifmm_gather_pack_f32": [_P, _P, _P, _P, _P, _I, _I, _P, _P, _P],
    "kifmm_gather_pack_f64": [_P, _P, _P, _P, _P, _I, _I, _P, _P, _P],
    "kifmm_gather_charges_f32": [_P, _P, _I, _I, _P, _P],
    "kifmm_gather_charges_f64": [_P, _P, _I, _I, _P, _P],
    "kifmm_split_tf32": [_P, _I, _P, _P, _P],
    "kifmm_m2l_sweep_tc_f32": [_P, _P, _P, _P, _I, _I, _P, _P, _P, _P, _I, _I, _I, _P, _P],
    "kifmm_chain_f32": [_I, _P, _I, _C, _I, _P, _I, _I, _C, _P, _P, _P, _I, _I, _I, _I, _I, _I,
                        _P, _P, _P, _D, _D, _D, _P, _I, _P, _C, _P],
    "kifmm_chain_f64": [_I, _P, _I, _C, _I, _P, _I, _I, _C, _P, _P, _P, _I, _I, _I, _I, _I, _I,
                        _P, _P, _P, _D, _D, _D, _P, _I, _P, _C, _P],
    "kifmm_dense_split_tf32": [_P, _P, _I, _I, _I, _I, _P, _P, _P],
    "kifmm_m2l_sweep_tma_f32": [_P, _P, _P, _P, _I, _I, _I, _P, _P, _I, _P, _P, _I, _I, _P, _P],
    "kifmm_m2l_sweep_tmem_f32": [_P, _P, _I, _I, _P, _P, _I, _P, _I, _P, _P, _I, _I, _I, _P, _P],
    "kifmm_m2l_sweep_tmem_splits": [_I, _I, _I, _P],
    "kifmm_m2l_sweep_tmem_trace": [_P, _I],
    "kifmm_scatter_add_rows_f32": [_P, _P, _I, _I, _P, _P],
    "kifmm_scatter_add_rows_f64": [_P, _P, _I, _I, _P, _P],
    "kifmm_p2p_mutual_f32": [_P, _P, _P, _I, _P, _I, _P, _P, _P, _I, _I, _C, _P, _P],
    "kifmm_p2p_mutual_f64": [_P, _P, _P, _I, _P, _I, _P, _P, _P, _I, _I, _C, _P, _P],
    "kifmm_p2p_mutual_reduce_f32": [_P, _P, _I, _I, _P, _P, _P, _I, _P, _P, _P],
    "kifmm_p2p_mutual_reduce_f64": [_P, _P, _I, _I, _P, _P, _P, _I, _P, _P, _P],
    "kifmm_p2p_mutual_grad_f32": [_P, _P, _P, _I, _P, _I, _P, _P, _P, _I, _I, _C, _P, _P],
    "kifmm_p2p_mutual_grad_f64": [_P, _P, _P, _I, _P, _I, _P, _P, _P, _I, _I, _C, _P, _P],
    "kifmm_p2p_mutual_reduce_grad_f32": [_P, _P, _I, _I, _P, _P, _P, _I, _P, _P, _P, _P],
    "kifmm_p2p_mutual_reduce_grad_f64": [_P, _P, _I, _I, _P, _P, _P, _I, _P, _P, _P, _P],
    "kifmm_sm_target": [],
    "kifmm_probe": [_C, _I, _I, _I, _P, _P],
}


class NativeError(RuntimeError):
    """A device entry point returned a nonzero status."""


_lib = None


def load():
    """Load the shared library (once) and declare every entry point."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build the CUDA library first "
                          "(python -c 'import __graft_entry__ as g; g.build()')")
    lib = ctypes.CDLL(LIB_PATH)
    for name, argtypes in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = ctypes.c_int
    _lib = lib
    return lib


def call(name: str, *args):
    st = getattr(load(), name)(*args)
    if st != 0:
        raise NativeError(f"{name} failed with status {st}")
    return st


def exported_symbols():
    return list(SIGNATURES)
