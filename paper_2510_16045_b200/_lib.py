"""ctypes binding of the C-ABI in ``include/amsq_b200.h`` (libamsq_b200.so).

Loading never silently degrades: a missing library raises ``ImportError`` telling the
user to build it, and every device entry point returns AMSQ_ENODEV (raised as
:class:`NoDeviceError`) when there is no sm_100a GPU.
"""
from __future__ import annotations

import ctypes as C
import os

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libamsq_b200.so")
# experiments only (tools/): load a variant build of the same library, e.g. build/variants/*.so
LIB_PATH = os.environ.get("AMSQ_LIB", LIB_PATH)

AMSQ_OK, AMSQ_EINVAL, AMSQ_ECORRUPT, AMSQ_ECUDA, AMSQ_ENCCL, AMSQ_ENOMEM, AMSQ_ENODEV = range(7)


class AmsqError(RuntimeError):
    """Base for runtime failures (std::runtime_error in the reference)."""


class CorruptError(AmsqError):
    pass


class CudaError(AmsqError):
    pass


class NcclError(AmsqError):
    pass


class NoDeviceError(AmsqError):
    pass


class SchemeInfo(C.Structure):
    _fields_ = [("id", C.c_int), ("exp_bits", C.c_int), ("man_bits", C.c_int), ("bias", C.c_int),
                ("k", C.c_int), ("block", C.c_size_t), ("words_per_block", C.c_size_t),
                ("name", C.c_char_p), ("device_supported", C.c_int)]


class WeightInfo(C.Structure):
    _fields_ = [("scheme_id", C.c_int), ("rows", C.c_size_t), ("cols", C.c_size_t),
                ("padded_cols", C.c_size_t), ("payload_bytes", C.c_size_t),
                ("device_bytes", C.c_size_t), ("row_tiles", C.c_size_t),
                ("k_tiles", C.c_size_t), ("device", C.c_int), ("n_groups", C.c_int),
                ("g_big", C.c_int), ("n_big", C.c_int), ("csplit", C.c_int)]


AMSQ_DTYPE_F16, AMSQ_DTYPE_BF16 = 0, 1

# Every symbol include/amsq_b200.h declares, with (restype, argtypes).
_P, _SZ, _I, _U16P, _U8P = C.c_void_p, C.c_size_t, C.c_int, C.c_void_p, C.c_void_p
SIGNATURES = {
    "amsq_last_error": (C.c_char_p, []),
    "amsq_version": (C.c_char_p, []),
    "amsq_scheme_info": (_I, [_I, C.POINTER(SchemeInfo)]),
    "amsq_scheme_by_name": (_I, [C.c_char_p, C.POINTER(C.c_int)]),
    "amsq_packed_payload_bytes": (_SZ, [_I, _SZ, _SZ]),
    "amsq_float_to_half": (C.c_uint16, [C.c_float]),
    "amsq_half_to_float": (C.c_float, [C.c_uint16]),
    "amsq_restore_table": (_I, [_I, _U16P, _SZ]),
    "amsq_pack_row": (_I, [_I, _U8P, _SZ, _U16P, _SZ]),
    "amsq_unpack_row": (_I, [_I, _U16P, _SZ, _U8P, _SZ]),
    "amsq_quantize_tensor": (_I, [_I, _SZ, _SZ, _P, _I, C.POINTER(_SZ), C.POINTER(_SZ), _U16P,
                                  _U16P]),
    "amsq_quantize_device": (_I, [_I, _P, _SZ, _SZ, _SZ, _P, _P, _SZ, _I, _P]),
    "amsq_quantize_device_host": (_I, [_I, _SZ, _SZ, _P, _I, C.POINTER(_SZ), C.POINTER(_SZ), _P, _P]),
    "amsq_container_size": (_I, [_I, _SZ, _SZ, C.POINTER(_SZ)]),
    "amsq_container_write": (_I, [_I, _SZ, _SZ, _SZ, _U16P, _U16P, _SZ, _U8P, _SZ]),
    "amsq_container_read": (_I, [_U8P, _SZ, C.POINTER(C.c_int), C.POINTER(_SZ), C.POINTER(_SZ),
                                 C.POINTER(_SZ), _U16P, _SZ, _U16P, _SZ]),
    "amsq_device_layout_bytes": (_SZ, [_I, _SZ, _SZ]),
    "amsq_device_layout_plan": (_I, [_I, _SZ, _SZ, _P]),
    "amsq_repack": (_I, [_I, _SZ, _SZ, _SZ, _U16P, _SZ, _U8P, _SZ]),
    "amsq_unrepack": (_I, [_I, _SZ, _SZ, _SZ, _U8P, _SZ, _U16P, _SZ]),
    "amsq_weight_upload": (_I, [_I, _SZ, _SZ, _SZ, _U16P, _U16P, _SZ, _I, _P, C.POINTER(_P)]),
    "amsq_weight_upload_rows": (_I, [_I, _SZ, _SZ, _SZ, _U16P, _U16P, _SZ, _SZ, _SZ, _I, _P,
                                     C.POINTER(_P)]),
    "amsq_weight_upload_container": (_I, [_U8P, _SZ, _SZ, _SZ, _I, _P, C.POINTER(_P)]),
    "amsq_weight_upload_file": (_I, [C.c_char_p, _SZ, _SZ, _I, _P, C.POINTER(_P)]),
    "amsq_weight_download": (_I, [_P, _U16P, _SZ, _U16P, _SZ]),
    "amsq_weight_clone": (_I, [_P, _P, C.POINTER(_P)]),
    "amsq_weight_free": (_I, [_P]),
    "amsq_weight_info": (_I, [_P, C.POINTER(WeightInfo)]),
    "amsq_restore_grid_f16": (_I, [_P, _P, _P]),
    "amsq_restore_f32": (_I, [_P, _P, _P]),
    "amsq_restore_f16": (_I, [_P, _P, _P]),
    "amsq_restore_to_host": (_I, [_P, _I, _P, _SZ, _P]),
    "amsq_linear": (_I, [_P, _P, _SZ, _P, _P]),
    "amsq_linear_chain": (_I, [_P, _P, _SZ, _P, _P, _P]),
    "amsq_debug_set_chain_prefetch": (_I, [_I]),
    "amsq_linear_ld": (_I, [_P, _P, _SZ, _P, _SZ, _P]),
    "amsq_linear_ex": (_I, [_P, _P, _I, _SZ, _P, _I, _SZ, _P]),
    "amsq_gemv_host": (_I, [_P, _U16P, _SZ, _SZ, _U16P, _P]),
    "amsq_linear_tp": (_I, [_P, _P, _SZ, _P, _P, _SZ, _P, _I, _P]),
    "amsq_linear_tp_group": (_I, [_I, _P, _P, _SZ, _P, _P, _SZ, _P, _P]),
    "amsq_tp_create_local": (_I, [_I, _P, _SZ, _P]),
    "amsq_tp_segment_create": (_I, [_I, _I, _I, _SZ, _P, C.POINTER(_P)]),
    "amsq_tp_attach": (_I, [_P, _P]),
    "amsq_tp_arena": (_I, [_P, C.POINTER(_P), C.POINTER(_SZ)]),
    "amsq_tp_error": (_I, [_P, C.POINTER(C.c_int)]),
    "amsq_tp_destroy": (_I, [_P]),
    "amsq_linear_tp_fused": (_I, [_P, _P, _P, _SZ, _SZ, _P]),
    "amsq_tp_unshard": (_I, [_P, _SZ, _SZ, _SZ, _P, _P]),
    "amsq_nccl_unique_id": (_I, [_P, _SZ]),
    "amsq_nccl_comm_init_rank": (_I, [_P, _SZ, _I, _I, _I, C.POINTER(_P)]),
    "amsq_nccl_comm_init_all": (_I, [_I, _P, _P]),
    "amsq_nccl_comm_destroy": (_I, [_P]),
    "amsq_kernel_launch_count": (C.c_uint64, []),
    "amsq_debug_set_trace": (None, [_P]),
    "amsq_debug_set_k3_min_batch": (_I, [_I]),
    "amsq_linear_uses_tc": (_I, [_I, _SZ]),
    "amsq_debug_set_k3_pair": (_I, [_I]),
    "amsq_debug_set_host_direct": (_I, [_I]),
}

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built: run `python __graft_entry__.py` "
                              "or `python -m paper_2510_16045_b200._build`")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            if "AMSQ_LIB" in os.environ and not hasattr(L, name):
                continue  # an older build loaded for A/B timing
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc == AMSQ_OK:
        return
    msg = lib().amsq_last_error().decode(errors="replace")
    full = f"{what}: {msg}" if what else msg
    if rc == AMSQ_EINVAL:
        raise ValueError(full)  # std::invalid_argument
    if rc == AMSQ_ECORRUPT:
        raise CorruptError(full)
    if rc == AMSQ_ENODEV:
        raise NoDeviceError(full)
    if rc == AMSQ_ENCCL:
        raise NcclError(full)
    if rc in (AMSQ_ECUDA, AMSQ_ENOMEM):
        raise CudaError(full)
    raise AmsqError(f"status {rc}: {full}")
