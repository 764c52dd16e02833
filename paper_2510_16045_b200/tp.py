"""Column-parallel (N-sharded) tensor parallelism of the AMS linear.

Output channels are independent in the reference (own scale, own word run,
quantize.hpp:57-60; per-row accumulation, kernels.hpp:161-184), so a rank's shard is a
zero-copy slice of whole payload rows plus ``scales[n0:n1]``. The sharded reference output
is exactly the matching slice of the full output. Rank p:

  1. holds rows [p*N/P, (p+1)*N/P)           (:func:`shard_range`, :func:`shard_tensor`)
  2. computes y_p = x W_p^T, [M][N/P]         (the K2 kernel, :meth:`ShardedLinear.forward`)
  3. all-gathers the shards over NCCL          -> [P][M][N/P]
  4. permutes to the reference layout [M][N]   (``amsq_tp_unshard`` kernel; host restatement
                                               :func:`unshard_host` for the tests)

``torch.distributed`` is the plumbing (one process per GPU, NCCL over NVLink); the C-ABI
also offers ``amsq_linear_tp`` for C++ hosts that own an ``ncclComm_t``.
"""
from __future__ import annotations

from typing import Optional

import numpy as np

from . import amsq
from ._lib import check, lib


def shard_range(rows: int, nranks: int, rank: int) -> tuple[int, int]:
    """(row0, nrows) of `rank`. N must split evenly (every Llama-3.1-70B N divides by 8):
    the all-gather exchanges equal-sized [M][N/P] shards."""
    if nranks < 1 or not 0 <= rank < nranks:
        raise ValueError(f"bad rank {rank} of {nranks}")
    if rows % nranks:
        raise ValueError(f"N={rows} does not split evenly over {nranks} ranks")
    n = rows // nranks
    return rank * n, n


def shard_tensor(qt: amsq.QuantizedTensor, nranks: int, rank: int) -> amsq.QuantizedTensor:
    """The rank's rows as a QuantizedTensor of its own (views of the reference stream)."""
    row0, n = shard_range(qt.rows, nranks, rank)
    wpr = qt.words_per_row()
    return amsq.QuantizedTensor(qt.scheme, n, qt.cols, qt.padded_cols, qt.scales[row0:row0 + n],
                                qt.payload[row0 * wpr:(row0 + n) * wpr])


def unshard_host(gathered: np.ndarray, nranks: int, batch: int, n_local: int) -> np.ndarray:
    """[P][M][n] -> [M][P*n]: the permutation amsq_tp_unshard applies on the device."""
    g = np.asarray(gathered).reshape(nranks, batch, n_local)
    return np.ascontiguousarray(g.transpose(1, 0, 2).reshape(batch, nranks * n_local))


class ShardedLinear:
    """One rank's shard of a column-parallel AMS linear, gathered with torch.distributed."""

    def __init__(self, qt: amsq.QuantizedTensor, group=None, device: Optional[int] = None):
        import torch
        import torch.distributed as dist

        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.device = torch.cuda.current_device() if device is None else device
        self.rows, self.cols = qt.rows, qt.cols
        self.row0, self.n_local = shard_range(qt.rows, self.world, self.rank)
        self.weight = amsq.DeviceWeight(qt, device=self.device, row0=self.row0,
                                        nrows=self.n_local)

    def forward(self, x, out=None):
        """x: [M][K] fp16 on this rank's GPU -> [M][N] fp16 (every rank gets the full output)."""
        import torch
        import torch.distributed as dist

        m = x.shape[0]
        local = self.weight.linear(x)  # [M][N/P]
        if self.world == 1:
            if out is not None:
                out.copy_(local)
                return out
            return local
        gathered = torch.empty(self.world * m * self.n_local, dtype=torch.float16,
                               device=x.device)
        dist.all_gather_into_tensor(gathered, local.reshape(-1), group=self.group)
        if out is None:
            out = torch.empty(m, self.rows, dtype=torch.float16, device=x.device)
        st = torch.cuda.current_stream(x.device).cuda_stream
        check(lib().amsq_tp_unshard(gathered.data_ptr(), self.world, m, self.n_local,
                                    out.data_ptr(), st), "amsq_tp_unshard")
        return out

    __call__ = forward


class FusedTPGroup:
    """Single-process fused column-parallel group (amsq_tp_create_local): rank r's shard of a
    weight runs amsq_linear_tp_fused, whose epilogue stores every output element into every
    rank's arena over NVLink; a device-side flag barrier replaces the NCCL all-gather and the
    unshard permutation. ``devices`` may repeat (virtual ranks on one GPU, for tests)."""

    def __init__(self, devices, arena_bytes: int):
        import ctypes as C
        self.devices = list(devices)
        self.nranks = len(self.devices)
        self.arena_bytes = int(arena_bytes)
        self._h = (C.c_void_p * self.nranks)()
        devs = (C.c_int * self.nranks)(*self.devices)
        check(lib().amsq_tp_create_local(self.nranks, devs, self.arena_bytes, self._h),
              "tp_create_local")

    def handle(self, rank: int) -> int:
        return self._h[rank]

    def arena(self, rank: int):
        """This rank's arena as a uint8 torch tensor view (device memory owned by the group)."""
        import ctypes as C
        import torch
        ptr, n = C.c_void_p(), C.c_size_t()
        check(lib().amsq_tp_arena(self._h[rank], C.byref(ptr), C.byref(n)), "tp_arena")
        return _device_view(ptr.value, n.value, self.devices[rank])

    def linear(self, rank: int, shard: amsq.DeviceWeight, x, y_offset: int = 0, stream=None):
        """Launch rank's fused linear on x ([M][K] fp16 on the rank's device)."""
        import torch
        st = stream.cuda_stream if stream is not None else \
            torch.cuda.current_stream(self.devices[rank]).cuda_stream
        check(lib().amsq_linear_tp_fused(shard.handle, self._h[rank], x.data_ptr(), x.shape[0],
                                         y_offset, st), "linear_tp_fused")

    def error(self, rank: int) -> int:
        import ctypes as C
        e = C.c_int(0)
        check(lib().amsq_tp_error(self._h[rank], C.byref(e)), "tp_error")
        return e.value

    def close(self):
        for r in range(self.nranks):
            if self._h[r]:
                lib().amsq_tp_destroy(self._h[r])
                self._h[r] = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _device_view(ptr: int, nbytes: int, device: int):
    """A torch uint8 tensor aliasing device memory the library owns (no copy, no free)."""
    import torch

    class _Arr:
        __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                    "version": 3, "strides": None}
    with torch.cuda.device(device):
        return torch.as_tensor(_Arr(), device=f"cuda:{device}")
