"""Python mirror of the reference's ``amsq::`` API over the B200 C-ABI.

Names, argument meaning and error behaviour follow
``/root/reference/proj/include/amsq`` (cited per function), so the parity tests read
like the reference's own tests: ``std::invalid_argument`` surfaces as ``ValueError``,
``std::runtime_error`` as :class:`CorruptError` (a ``RuntimeError``).

Host-side pieces (scheme tables, pack/unpack, the quantizer, the container) run in the
C++ core of ``libamsq_b200.so``. The hot path -- restore and the fused linear -- runs
only on the sm_100a kernels: :func:`gemv`, :func:`restore_matrix` and friends upload to
the GPU and raise :class:`NoDeviceError` when there is none. There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from ._lib import CorruptError, NoDeviceError, check, lib  # noqa: F401  (re-exported)


# ------------------------------------------------------------------ schemes
@dataclass(frozen=True)
class QuantScheme:
    """scheme.hpp:32-56 QuantScheme + packing.hpp:51-63 block geometry."""

    id: int
    name: str
    exp_bits: int
    man_bits: int
    bias: int
    k: int
    block: int
    words_per_block: int
    device_supported: bool

    def effective_bits(self) -> float:  # scheme.hpp:38-41
        b = 1 + self.exp_bits + self.man_bits
        return (b - 1) + 1.0 / self.k if self.k > 1 else float(b)

    def bits_label(self) -> str:  # scheme.hpp:44-51
        b = 1 + self.exp_bits + self.man_bits
        if self.k == 1:
            return str(b)
        frac = str(100 // self.k)
        if frac.endswith("0"):
            frac = frac[:-1]
        return f"{b - 1}.{frac}"

    @property
    def code_count(self) -> int:
        return 1 << (1 + self.exp_bits + self.man_bits)

    @property
    def sign_mask(self) -> int:
        return 1 << (self.exp_bits + self.man_bits)


_SCHEMES: Optional[list] = None


def all_schemes() -> list:
    """scheme.hpp:59-74 -- the eight shipped schemes, indexed by id."""
    global _SCHEMES
    if _SCHEMES is None:
        out = []
        for i in range(8):
            info = _lib.SchemeInfo()
            check(lib().amsq_scheme_info(i, C.byref(info)), "scheme_info")
            out.append(QuantScheme(info.id, info.name.decode(), info.exp_bits, info.man_bits,
                                   info.bias, info.k, int(info.block), int(info.words_per_block),
                                   bool(info.device_supported)))
        _SCHEMES = out
    return _SCHEMES


def scheme_by_id(i: int) -> QuantScheme:
    """scheme.hpp:76-82 (ValueError for unknown ids, like std::invalid_argument)."""
    if not 0 <= int(i) < 8:
        raise ValueError(f"unknown scheme id {i}")
    return all_schemes()[int(i)]


def scheme_by_name(name: str) -> QuantScheme:
    """scheme.hpp:84-89."""
    sid = C.c_int(-1)
    check(lib().amsq_scheme_by_name(name.encode(), C.byref(sid)), "scheme_by_name")
    return all_schemes()[sid.value]


def _sid(scheme) -> int:
    return scheme.id if isinstance(scheme, QuantScheme) else int(scheme)


# ------------------------------------------------------------------ binary16 / format
def float_to_half(f: float) -> int:
    """half.hpp:65-67 (RNE, overflow to inf)."""
    return int(lib().amsq_float_to_half(float(f)))


def half_to_float(h: int) -> float:
    """half.hpp:69-71 (exact)."""
    return float(lib().amsq_half_to_float(int(h)))


def restore_table(scheme) -> np.ndarray:
    """format.hpp:196-198 restore_table: binary16 pattern per raw code."""
    s = scheme_by_id(_sid(scheme))
    out = np.zeros(s.code_count, np.uint16)
    check(lib().amsq_restore_table(s.id, out.ctypes.data, out.size), "restore_table")
    return out


def to_fp16_bits(code: int, scheme) -> int:
    """format.hpp:190-192."""
    return int(restore_table(scheme)[code])


def packed_payload_bytes(scheme, rows: int, cols: int) -> int:
    """quantize.hpp:64-69."""
    return int(lib().amsq_packed_payload_bytes(_sid(scheme), rows, cols))


def round_up(n: int, multiple: int) -> int:
    """matrix.hpp:42-44."""
    return (n + multiple - 1) // multiple * multiple


# ------------------------------------------------------------------ codec
def pack_row(codes, scheme) -> np.ndarray:
    """packing.hpp:216-239 (ValueError on length, CorruptError on a shared-bit mismatch)."""
    s = scheme_by_id(_sid(scheme))
    codes = np.ascontiguousarray(codes, np.uint8)
    words = np.zeros(codes.size // s.block * s.words_per_block, np.uint16)
    check(lib().amsq_pack_row(s.id, codes.ctypes.data, codes.size, words.ctypes.data, words.size),
          "pack_row")
    return words


def unpack_row(words, scheme) -> np.ndarray:
    """packing.hpp:243-266."""
    s = scheme_by_id(_sid(scheme))
    words = np.ascontiguousarray(words, np.uint16)
    codes = np.zeros(words.size // s.words_per_block * s.block, np.uint8)
    check(lib().amsq_unpack_row(s.id, words.ctypes.data, words.size, codes.ctypes.data,
                                codes.size), "unpack_row")
    return codes


# ------------------------------------------------------------------ tensors
@dataclass
class QuantizedTensor:
    """quantize.hpp:45-61: payload words row after row, one binary16 scale per row."""

    scheme: QuantScheme
    rows: int
    cols: int
    padded_cols: int
    scales: np.ndarray = field(repr=False)
    payload: np.ndarray = field(repr=False)

    def words_per_row(self) -> int:
        return 0 if self.rows == 0 else self.payload.size // self.rows

    def payload_bytes(self) -> int:
        return self.payload.size * 2

    def row_words(self, r: int) -> np.ndarray:
        w = self.words_per_row()
        return self.payload[r * w:(r + 1) * w]


def quantize_tensor(weights, scheme, threads: int = 1) -> QuantizedTensor:
    """quantize.hpp:188-216: pad, RTN, Adaptive Searching (k > 1), pack -- on the host."""
    s = scheme_by_id(_sid(scheme))
    w = np.ascontiguousarray(weights, np.float32)
    if w.ndim != 2 or w.size == 0:
        raise ValueError("quantize_tensor: empty matrix")
    rows, cols = w.shape
    pc, nw = C.c_size_t(0), C.c_size_t(0)
    check(lib().amsq_quantize_tensor(s.id, rows, cols, None, threads, C.byref(pc), C.byref(nw),
                                     None, None), "quantize_tensor")
    scales = np.zeros(rows, np.uint16)
    payload = np.zeros(nw.value, np.uint16)
    check(lib().amsq_quantize_tensor(s.id, rows, cols, w.ctypes.data, threads, C.byref(pc),
                                     C.byref(nw), scales.ctypes.data, payload.ctypes.data),
          "quantize_tensor")
    return QuantizedTensor(s, rows, cols, pc.value, scales, payload)


def quantize_tensor_device(weights, scheme, device: int = 0, stream=None,
                           to_host: bool = True):
    """quantize_tensor on the GPU (amsq_quantize_device): bit-identical
    scales and payload. `weights` is a CUDA float32 [rows][cols] tensor (or array-like, moved
    to `device`). Returns a QuantizedTensor (host arrays) or, with to_host=False, the device
    tensors (scales u16 as int16, payload u16 as int16) plus padded_cols."""
    import torch
    s = scheme_by_id(_sid(scheme))
    w = torch.as_tensor(weights, dtype=torch.float32, device=f"cuda:{device}")
    if w.ndim != 2 or w.numel() == 0:
        raise ValueError("quantize_tensor: empty matrix")
    w = w.contiguous()
    rows, cols = w.shape
    pc, nw = C.c_size_t(0), C.c_size_t(0)
    check(lib().amsq_quantize_tensor(s.id, rows, cols, None, 1, C.byref(pc), C.byref(nw),
                                     None, None), "quantize_tensor")
    sc = torch.empty(rows, dtype=torch.int16, device=w.device)
    pl = torch.empty(nw.value, dtype=torch.int16, device=w.device)
    check(lib().amsq_quantize_device(s.id, w.data_ptr(), rows, cols, cols, sc.data_ptr(),
                                     pl.data_ptr(), nw.value, device,
                                     _stream_ptr(stream, device)), "quantize_device")
    if not to_host:
        return sc, pl, pc.value
    return QuantizedTensor(s, rows, cols, pc.value, sc.cpu().numpy().view(np.uint16).copy(),
                           pl.cpu().numpy().view(np.uint16).copy())


# ------------------------------------------------------------------ container
def write_amsq(qt: QuantizedTensor) -> bytes:
    """container.hpp:63-77 (returns the bytes instead of writing a stream)."""
    n = C.c_size_t(0)
    check(lib().amsq_container_size(qt.scheme.id, qt.rows, qt.cols, C.byref(n)), "container_size")
    out = np.zeros(n.value, np.uint8)
    check(lib().amsq_container_write(qt.scheme.id, qt.rows, qt.cols, qt.padded_cols,
                                     np.ascontiguousarray(qt.scales).ctypes.data,
                                     np.ascontiguousarray(qt.payload).ctypes.data,
                                     qt.payload.size, out.ctypes.data, out.size), "write_amsq")
    return out.tobytes()


def read_amsq(data: bytes) -> QuantizedTensor:
    """container.hpp:79-115 validating reader."""
    buf = np.frombuffer(data, np.uint8)
    sid, rows, cols, pc = C.c_int(0), C.c_size_t(0), C.c_size_t(0), C.c_size_t(0)
    check(lib().amsq_container_read(buf.ctypes.data, buf.size, C.byref(sid), C.byref(rows),
                                    C.byref(cols), C.byref(pc), None, 0, None, 0), "read_amsq")
    s = scheme_by_id(sid.value)
    scales = np.zeros(rows.value, np.uint16)
    payload = np.zeros(rows.value * (pc.value // s.block) * s.words_per_block, np.uint16)
    check(lib().amsq_container_read(buf.ctypes.data, buf.size, None, None, None, None,
                                    scales.ctypes.data, scales.size, payload.ctypes.data,
                                    payload.size), "read_amsq")
    return QuantizedTensor(s, rows.value, cols.value, pc.value, scales, payload)


def save_amsq(path: str, qt: QuantizedTensor) -> None:
    with open(path, "wb") as f:
        f.write(write_amsq(qt))


def load_amsq(path: str) -> QuantizedTensor:
    with open(path, "rb") as f:
        return read_amsq(f.read())


# ------------------------------------------------------------------ device weights
def _stream_ptr(stream, device: Optional[int] = None) -> Optional[int]:
    """The raw cudaStream_t: `stream` itself, or torch's current stream OF `device` (the
    library switches to the weight's device, and a stream of another device cannot launch
    there)."""
    if stream is None:
        import torch
        dev = torch.cuda.current_device() if device is None else device
        return torch.cuda.current_stream(dev).cuda_stream
    return stream if isinstance(stream, int) else stream.cuda_stream


class DeviceWeight:
    """A QuantizedTensor uploaded into the sm_100a tile layout (immutable, owns its memory).

    ``row0``/``nrows`` select an N-shard for column-parallel tensor parallelism.
    """

    def __init__(self, qt: QuantizedTensor, device: int = 0, stream=None, row0: int = 0,
                 nrows: Optional[int] = None):
        self._h = C.c_void_p(None)
        nrows = qt.rows - row0 if nrows is None else nrows
        st = _stream_ptr(stream, device) if _torch_cuda_ok() else None
        check(lib().amsq_weight_upload_rows(
            qt.scheme.id, qt.rows, qt.cols, qt.padded_cols,
            np.ascontiguousarray(qt.scales).ctypes.data,
            np.ascontiguousarray(qt.payload).ctypes.data, qt.payload.size, row0, nrows, device,
            st, C.byref(self._h)), "weight_upload")
        self.scheme = qt.scheme
        self.rows, self.cols, self.padded_cols = nrows, qt.cols, qt.padded_cols
        self.device = device
        info = self.info()
        self.device_bytes = int(info.device_bytes)
        self.payload_bytes = int(info.payload_bytes)

    @classmethod
    def from_container(cls, data: bytes, device: int = 0, row0: int = 0, nrows: int = 0):
        self = cls.__new__(cls)
        self._h = C.c_void_p(None)
        buf = np.frombuffer(data, np.uint8)
        check(lib().amsq_weight_upload_container(buf.ctypes.data, buf.size, row0, nrows, device,
                                                 None, C.byref(self._h)), "upload_container")
        info = self.info()
        self.scheme = scheme_by_id(info.scheme_id)
        self.rows, self.cols, self.padded_cols = int(info.rows), int(info.cols), int(info.padded_cols)
        self.device = device
        self.device_bytes = int(info.device_bytes)
        self.payload_bytes = int(info.payload_bytes)
        return self

    @classmethod
    def from_file(cls, path: str, device: int = 0, row0: int = 0, nrows: int = 0):
        """An AMSQ container file, mmap'd and uploaded (only rows [row0, row0+nrows) are
        read; container.hpp:79-115 validation)."""
        self = cls.__new__(cls)
        self._h = C.c_void_p(None)
        check(lib().amsq_weight_upload_file(os.fsencode(path), row0, nrows, device, None,
                                            C.byref(self._h)), "upload_file")
        info = self.info()
        self.scheme = scheme_by_id(info.scheme_id)
        self.rows, self.cols, self.padded_cols = int(info.rows), int(info.cols), int(info.padded_cols)
        self.device = device
        self.device_bytes = int(info.device_bytes)
        self.payload_bytes = int(info.payload_bytes)
        return self

    @property
    def handle(self) -> int:
        return self._h.value

    def info(self) -> _lib.WeightInfo:
        out = _lib.WeightInfo()
        check(lib().amsq_weight_info(self._h, C.byref(out)), "weight_info")
        return out

    def download(self) -> QuantizedTensor:
        """Inverse repack: the reference payload words, bit-exact."""
        scales = np.zeros(self.rows, np.uint16)
        payload = np.zeros(self.rows * (self.padded_cols // self.scheme.block) *
                           self.scheme.words_per_block, np.uint16)
        check(lib().amsq_weight_download(self._h, scales.ctypes.data, scales.size,
                                         payload.ctypes.data, payload.size), "weight_download")
        return QuantizedTensor(self.scheme, self.rows, self.cols, self.padded_cols, scales, payload)

    # --- device-tensor API (torch tensors for memory; fp16 views as uint16 bits are fine)
    def restore_grid(self, out=None, stream=None):
        import torch
        if out is None:
            out = torch.empty((self.rows, self.padded_cols), dtype=torch.float16,
                              device=f"cuda:{self.device}")
        check(lib().amsq_restore_grid_f16(self._h, out.data_ptr(), _stream_ptr(stream, self.device)),
              "restore_grid")
        return out

    def restore_f32(self, out=None, stream=None):
        import torch
        if out is None:
            out = torch.empty((self.rows, self.cols), dtype=torch.float32,
                              device=f"cuda:{self.device}")
        check(lib().amsq_restore_f32(self._h, out.data_ptr(), _stream_ptr(stream, self.device)), "restore_f32")
        return out

    def restore_f16(self, out=None, stream=None):
        import torch
        if out is None:
            out = torch.empty((self.rows, self.cols), dtype=torch.float16,
                              device=f"cuda:{self.device}")
        check(lib().amsq_restore_f16(self._h, out.data_ptr(), _stream_ptr(stream, self.device)), "restore_f16")
        return out

    def linear(self, x, out=None, stream=None):
        """y[M][rows] = x[M][cols] @ W^T, fp32 accumulation; x and y fp16 (the reference's
        dtype) or bf16 (amsq_linear_ex: exact power-of-two staging through fp16)."""
        import torch
        if x.dim() != 2 or x.shape[1] != self.cols or x.dtype not in (torch.float16,
                                                                      torch.bfloat16):
            raise ValueError("gemv: activation shape mismatch")
        x = x.contiguous()
        if out is None:
            out = torch.empty((x.shape[0], self.rows), dtype=x.dtype, device=x.device)
        elif out.dtype != x.dtype:
            raise ValueError("linear: out dtype must match x")
        st = _stream_ptr(stream, self.device)
        if x.dtype == torch.float16:
            check(lib().amsq_linear(self._h, x.data_ptr(), x.shape[0], out.data_ptr(), st),
                  "linear")
        else:
            check(lib().amsq_linear_ex(self._h, x.data_ptr(), _lib.AMSQ_DTYPE_BF16, x.shape[0],
                                       out.data_ptr(), _lib.AMSQ_DTYPE_BF16, out.stride(0), st),
                  "linear")
        return out

    def gemv_host(self, x: np.ndarray, batch: int, stream=None) -> np.ndarray:
        """Host fp16 bits in/out through amsq_gemv_host (H2D + kernel + D2H)."""
        x = np.ascontiguousarray(x, np.uint16).reshape(-1)
        y = np.zeros(batch * self.rows, np.uint16)
        st = _stream_ptr(stream, self.device) if _torch_cuda_ok() else None
        check(lib().amsq_gemv_host(self._h, x.ctypes.data, x.size, batch, y.ctypes.data, st),
              "gemv")
        return y

    def clone(self, stream=None) -> "DeviceWeight":
        """An independent device copy (device-to-device; no host round trip)."""
        out = DeviceWeight.__new__(DeviceWeight)
        out._h = C.c_void_p(None)
        check(lib().amsq_weight_clone(self._h, _stream_ptr(stream, self.device), C.byref(out._h)),
              "clone")
        for k in ("scheme", "rows", "cols", "padded_cols", "device", "device_bytes", "payload_bytes"):
            if hasattr(self, k):
                setattr(out, k, getattr(self, k))
        return out

    def free(self):
        if self._h and self._h.value:
            lib().amsq_weight_free(self._h)
            self._h = C.c_void_p(None)

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _torch_cuda_ok() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


# ------------------------------------------------------------------ reference call shapes
def gemv(qt: QuantizedTensor, x, batch: int, threads: int = 1, device: int = 0) -> np.ndarray:
    """kernels.hpp:151-187 ``gemv(qt, x, batch, threads)`` computed on the GPU.

    ``x`` is fp16 bits ``[batch*cols]``; returns fp16 bits ``[batch*rows]``. ``threads``
    is accepted for signature parity and ignored.
    """
    x = np.ascontiguousarray(x, np.uint16).reshape(-1)
    if batch == 0 or x.size != batch * qt.cols:
        raise ValueError("gemv: activation shape mismatch")  # kernels.hpp:137-143
    w = DeviceWeight(qt, device=device)
    try:
        return w.gemv_host(x, batch)
    finally:
        w.free()


def restore_matrix(qt: QuantizedTensor, threads: int = 1, device: int = 0) -> np.ndarray:
    """kernels.hpp:100-124 on the GPU: fp32 ``w*s`` for the logical columns."""
    import torch
    w = DeviceWeight(qt, device=device)
    try:
        return w.restore_f32().cpu().numpy()
    finally:
        w.free()


def restore_matrix_half(qt: QuantizedTensor, threads: int = 1, device: int = 0) -> np.ndarray:
    """kernels.hpp:127-133 on the GPU: fp16 bits of ``w*s``."""
    import torch
    w = DeviceWeight(qt, device=device)
    try:
        return w.restore_f16().cpu().view(torch.int16).numpy().view(np.uint16)
    finally:
        w.free()


def restore_grid(qt: QuantizedTensor, device: int = 0) -> np.ndarray:
    """restore_block (kernels.hpp:55-63) over every padded column, on the GPU."""
    import torch
    w = DeviceWeight(qt, device=device)
    try:
        return w.restore_grid().cpu().view(torch.int16).numpy().view(np.uint16)
    finally:
        w.free()


def kernel_launch_count() -> int:
    return int(lib().amsq_kernel_launch_count())
