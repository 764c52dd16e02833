"""B200-native (sm_100a) AMS-Quant weight-only quantized linear.

Drop-in for the hot path of the reference toolkit (``amsq::quantize/pack/unpack/
restore/gemv``, /root/reference/proj/include/amsq): FP4.25-e2m2 (k=4) and
FP5.33-e2m3 (k=3) weights restored in registers and fed to the tensor cores.
See DESIGN.md for the layout and kernels, INTEGRATION.md for the C-ABI.
"""
from .amsq import (  # noqa: F401
    DeviceWeight,
    QuantizedTensor,
    QuantScheme,
    all_schemes,
    float_to_half,
    gemv,
    half_to_float,
    kernel_launch_count,
    load_amsq,
    pack_row,
    packed_payload_bytes,
    quantize_tensor,
    quantize_tensor_device,
    read_amsq,
    restore_grid,
    restore_matrix,
    restore_matrix_half,
    restore_table,
    round_up,
    save_amsq,
    scheme_by_id,
    scheme_by_name,
    to_fp16_bits,
    unpack_row,
    write_amsq,
)
from ._lib import AmsqError, CorruptError, CudaError, NcclError, NoDeviceError  # noqa: F401

__all__ = [n for n in dir() if not n.startswith("_")]
