"""ctypes binding of libmcf.so (the C-ABI in include/mcf.h).

The product path has no CPU fallback: if the shared library is missing or a
CUDA device is absent, every device entry point raises ``DeviceError``.
"""
from __future__ import annotations

import ctypes
import os

from .errors import DeviceError

_HERE = os.path.dirname(os.path.abspath(__file__))
# MCF_LIB: an alternative build of the same library (kernel A/B experiments)
LIB_PATH = os.environ.get("MCF_LIB") or os.path.join(_HERE, "libmcf.so")
_LIB = None

c_int, c_i32, c_i64, c_f32, c_size = ctypes.c_int, ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_size_t
vp = ctypes.c_void_p

# name -> (restype, argtypes); mirrors include/mcf.h one for one
SIGNATURES = {
    "mcf_version": (c_int, []),
    "mcf_last_error": (ctypes.c_char_p, []),
    "mcf_factor_ld": (c_int, [c_int]),
    "mcf_max_dim": (c_int, []),
    "mcf_csr_workspace_bytes": (c_size, [c_i64, c_i32]),
    "mcf_csr_build": (c_int, [vp, vp, vp, c_i64, c_i32, vp, vp, vp, vp, vp, c_size, vp]),
    "mcf_als_plan_bytes": (c_size, [c_i32, c_i64, c_i32]),
    "mcf_als_plan": (c_int, [vp, vp, c_i32, c_i32, c_i32, c_i64, vp, c_size,
                             ctypes.POINTER(c_i64), vp]),
    "mcf_als_workspace_bytes": (c_size, [c_i32, c_i64, c_i32]),
    "mcf_als_workspace_bytes_fixed": (c_size, [c_i32, c_i64, c_i32, c_i64, c_i64]),
    "mcf_als_half_step": (c_int, [vp, vp, vp, vp, vp, c_i64, vp, c_i32, c_f32, c_f32, c_f32, vp, vp,
                                  c_f32, vp, c_i32, c_i32, c_i32, vp, ctypes.POINTER(c_i64), vp,
                                  vp, vp, c_size, vp]),
    "mcf_als_half_step_bias": (c_int, [vp, vp, vp, vp, vp, c_i64, vp, c_i32, c_f32, c_f32, c_f32, vp,
                                       vp, c_f32, vp, c_i32, c_i32, c_i32, vp,
                                       ctypes.POINTER(c_i64), vp, vp, c_size, c_i32, c_f32, c_f32,
                                       vp]),
    "mcf_als_half_step_peers": (c_int, [vp, vp, vp, vp, vp, c_i64, vp, c_i32, c_f32, c_f32, c_f32,
                                        vp, vp, c_f32, vp, c_i32, c_i32, c_i32, vp,
                                        ctypes.POINTER(c_i64), vp, vp, vp, c_size, vp, c_i32,
                                        vp]),
    "mcf_als_half_step_multicast": (c_int, [vp, vp, vp, vp, vp, c_i64, vp, c_i32, c_f32, c_f32,
                                            c_f32, vp, vp, c_f32, vp, c_i32, c_i32, c_i32, vp,
                                            ctypes.POINTER(c_i64), vp, vp, vp, c_size, vp, vp]),
    "mcf_comm_id_bytes": (c_size, []),
    "mcf_comm_get_unique_id": (c_int, [vp, c_size]),
    "mcf_comm_init": (c_int, [vp, c_size, c_i32, c_i32, ctypes.POINTER(vp)]),
    "mcf_comm_destroy": (c_int, [vp]),
    "mcf_allgather_rows": (c_int, [vp, vp, c_i32, ctypes.POINTER(c_i64), ctypes.POINTER(c_i64),
                                   vp]),
    "mcf_mfitr_fixed": (c_int, [vp, vp, vp, c_i64, c_i32, vp, vp]),
    "mcf_mfitr_sgd_epoch": (c_int, [vp, vp, vp, vp, c_i32, vp, vp, vp, vp, vp, vp, vp, vp, c_f32,
                                    c_i32, c_f32, c_f32, c_f32, vp, vp, vp, c_i64, c_f32, c_f32,
                                    c_i32, vp]),
    "mcf_mfitr_sgd_epoch_locked": (c_int, [vp, vp, vp, vp, c_i32, vp, vp, vp, vp, vp, vp, vp, vp,
                                           c_f32, c_i32, c_f32, c_f32, c_f32, vp, vp, vp, c_i64,
                                           c_f32, c_f32, c_i32, vp, vp]),
    "mcf_lock_stress": (c_int, [vp, vp, c_i32, c_i32, c_i32, vp]),
    "mcf_als_half_step_mfitr": (c_int, [vp, vp, vp, vp, c_i64, vp, c_i32, c_f32, c_f32, vp, vp,
                                        c_f32, vp, c_i32, c_i32, vp, vp, vp, vp, c_size, c_f32, vp,
                                        vp, vp, c_i32, vp]),
    "mcf_mfitr_fixed_bsub": (c_int, [vp, vp, vp, c_i64, c_i32, vp, vp]),
    "mcf_mfitr_artist_workspace_bytes": (c_size, [c_i32]),
    "mcf_mfitr_artist_step": (c_int, [vp, vp, vp, c_i32, vp, vp, vp, vp, c_i32, c_f32, c_f32, vp,
                                      vp, c_size, vp]),
    "mcf_mfitr_targets": (c_int, [c_i32, vp, vp, vp, vp, c_i32, vp, vp, vp, vp, c_f32, c_i32, vp,
                                  vp]),
    "mcf_taxonomy_terms": (c_int, [vp, vp, vp, vp, vp, c_i32, c_i32, vp, c_i32, vp, vp, vp]),
    "mcf_edge_weights_workspace_bytes": (c_size, [c_i64, c_i32, c_i32]),
    "mcf_edge_weights": (c_int, [vp, vp, vp, c_i32, c_i32, vp, vp, c_i64, vp, vp, c_size, vp]),
    "mcf_predict_workspace_bytes": (c_size, [c_i64]),
    "mcf_predict_sse": (c_int, [vp, vp, vp, c_i64, vp, c_i32, vp, c_i32, c_i32, c_f32, vp, vp,
                                vp, vp, vp, c_f32, c_f32, vp, vp, vp, c_size, vp]),
    "mcf_sq_norms": (c_int, [vp, c_i32, c_i32, vp, vp, vp, c_size, vp]),
    "mcf_add_gathered": (c_int, [vp, vp, vp, c_i32, c_i32, vp, vp]),
}


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceError(f"{LIB_PATH} is not built; run `make` or "
                              "`python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().mcf_last_error().decode(errors="replace")
        raise DeviceError(f"{what} failed ({rc}): {msg}")


def ptr(t) -> int | None:
    """Device address of a tensor (None for None)."""
    return None if t is None else t.data_ptr()


def factor_ld(D: int) -> int:
    return (D + 3) // 4 * 4 if D <= 4 else (D + 7) // 8 * 8
