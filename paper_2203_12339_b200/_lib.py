"""ctypes binding of the sm_100a C ABI (include/sss_b200.h).

The product path has no CPU fallback: if the shared library is missing or
CUDA is unavailable, every entry point raises. The library is built in-tree
(``python -m paper_2203_12339_b200.build``) so it travels with the repo.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import torch

_SO = Path(__file__).resolve().parent / "_sss_b200.so"
_lib = None

_P = C.c_void_p
_I = C.c_int
_D = C.c_double

_SIGS = {
    "sss_haar2d": [_P, _P, _I, _I, _I, _I, _P],
    "sss_select_topn": [_P, _I, _I, _I, _P, _P, _P, _P, _P],
    "sss_select_topn_pack": [_P, _I, _I, _P, _P, _P, _P, _P, _P, _P],
    "sss_sh_irradiance": [_P, _P, _I, _I, _I, _P, _P, _P],
    "sss_env_project": [_P, _I, _I, _P, _P, _P, _P, _P, _P],
    "sss_env_irradiance": [_P, _I, _P, _P, _P, _I, _I, _I, _P, _P, _P],
    "sss_env_irradiance_sel": [_P, _I, _P, _P, _I, _I, _I, _P, _P, _P],
    "sss_env_transfer": [_P, _I, _P, _P, _I, _P, _P],
    "sss_material_weights": [_P, _P, _I, _I, _P, _P, _P],
    "sss_pack_x_bits": [_P, _I, _P, _P, _P],
    "sss_sweep_basis": [_I, _I, _I, _P, _P, _P],
    "sss_material_weights_batch": [_P, _P, _I, _I, _I, _P, _P, _P, _P, _P],
    "sss_sweep_gemm": [_I, _I, _P, _P, _P, C.c_float, C.c_float, _P, _P, _P, _P, _P],
    "sss_visibility": [_I, _P, _P, _I, _P, C.c_double, C.c_double, _P, _P, _P, _P],
    "sss_fold_weights": [_P, _I, _P, _P, _I, _P, C.c_double, _P, _P],
    "sss_transpose_f64": [_P, _I, _I, _P, _P, _P],
    "sss_fold_spmm": [_I, _I, _P, _P, _P, _P, _P, _P],
    "sss_fold_select": [_P, _I, _I, C.c_double, _P, _P, _P, _P, _P, _P, _P],
    "sss_fold_emit": [_P, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P],
    "sss_transfer_kfr": [_I, _I, C.c_uint, C.c_uint, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                         _P, _P, _P, _I, _I, _I, _P],
    "sss_transfer_flat16": [_I, _I, _P, _P, C.c_ulonglong, _P, _P, _P, _P, _I, _I, _I, _I, _I, _P,
                            _P, _P, _P, _I, _P, _P, _P],
    "sss_fold_apply_rows": [_I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P],
    "sss_fold_apply": [_I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "sss_direct_irradiance": [_I, _P, _P, _I, _P, _P, _P, C.c_double, C.c_double, _P, _P, _P, _P],
    "sss_direct_irradiance64": [_I, _P, _P, _I, _P, _P, _P, C.c_double, C.c_double, _P, _P, _P,
                                _P],
    "sss_edit_finish": [_I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "sss_edit_finish_wide": [_I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "sss_pair_block": [_I, _I, _I, _P, _P, _P, _P, _P, _I, _I, _P, _P, _I, C.c_float, _P, _P, _P],
    "sss_pair_rows_exact": [_I, _I, _P, _P, _I, _P, _P, _I, C.c_float, _I, _I, _P, _P],
    "sss_step1_select": [_P, _I, _I, _I, _P, _P, _P],
    "sss_step1_rows": [_P, _I, _P, _I, _I, _P, _P, _P],
    "sss_step2_select": [_P, _I, _D, _P, _P, _P, _P, _P, _P, _P, _P],
    "sss_emit": [_I, _P, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P],
    "sss_scan_u32": [_P, _P, C.c_size_t, _P, _P, _P],
    "sss_rowptr": [_P, _I, _I, C.c_uint64, _P, _P, _P],
    "sss_raster_fill": [_P, _I, _P, _P, _P, _P, _P, _I, _I, _P, _P, _P, _P, _D, _P, _P],
    "sss_raster_clear": [_I, _I, _D, _D, _D, _P, _P, _P],
    "sss_project_vertices": [_P, _I, _P, _D, _D, _I, _I, _P, _P, _P, _P, _P],
    "sss_vertex_colors": [_P, _P, _I, _P, _P],
    "sss_zero": [_P, C.c_ulonglong, _P],
    "sss_widen_frame": [_P, _P, C.c_longlong, _P, _P],
    "sss_encode_srgb8": [_P, C.c_longlong, _D, _P, _P],
    "sss_frame_replay": [_P, _I, _P, _P, _P, _P, _P, _P, _P, C.c_longlong, _P, _P, _P, _P,
                         C.c_ulonglong, _P],
    "sss_wavelet2d": [_P, _P, _I, _I, _I, _I, _I, _P],
    "sss_csr_apply": [_I, _P, _P, _P, _P, _P, _P, _P],
    "sss_transfer_rows": [_I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P],
    "sss_atlas_scatter": [_P, _I, _I, _P, _I, _P, _P],
    "sss_atlas_recombine": [_I, _I, _P, _P, _P, _P, _P],
    "sss_atlas_shade": [_I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "sss_energy_cut": [_P, _I, _I, _D, _P, _P, _P],
    "sss_bvh_any_hit": [_I, _P, _P, _P, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P],
}


class SSSError(RuntimeError):
    pass


def exported_symbols():
    return sorted(_SIGS) + ["sss_last_error", "sss_version"]


def load(require_cuda: bool = True):
    """Load the library (and bind signatures). Raises if it is missing."""
    global _lib
    if require_cuda and not torch.cuda.is_available():
        raise SSSError("CUDA device required: the relight path runs only on sm_100a")
    if _lib is not None:
        return _lib
    if not _SO.exists():
        raise SSSError(f"{_SO.name} is not built: run `python -m paper_2203_12339_b200.build` "
                       "(there is no CPU fallback)")
    lib = C.CDLL(str(_SO))
    lib.sss_last_error.restype = C.c_char_p
    lib.sss_version.restype = C.c_int
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
    _lib = lib
    return lib


def ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def stream_ptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def call(name, *args):
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        raise SSSError(f"{name} failed ({rc}): {lib.sss_last_error().decode()}")
