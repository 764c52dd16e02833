"""Column-parallel TP host logic, world size 2 over gloo on CPU.

Each rank takes its row shard (paper_2510_16045_b200.tp.shard_tensor), computes its
[M][N/P] output, all-gathers, and un-shards to [M][N]. The result must equal the
full single-device reference output bit for bit, because a row shard of the reference
stream produces exactly the matching slice of the reference output. On CPU the local
compute is the oracle (test infrastructure); the device path (K2 + amsq_tp_unshard) is
covered by the GPU test at the bottom.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_16045_b200 import tp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, sid, rows, cols, batch, result_dir):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from helpers import gaussian_x, quantized_gaussian
    from oracle import COracle
    orc = COracle()
    qt = quantized_gaussian(sid, rows, cols, seed=5)  # same bytes on every rank
    x = gaussian_x(batch, cols, seed=6)
    shard = tp.shard_tensor(qt, world, rank)
    y_local = orc.gemv(sid, shard.rows, cols, qt.padded_cols, shard.scales, shard.payload, x,
                       batch)  # [M][N/P] fp16 bits
    # gloo has no 16-bit integer collectives: the fp16 bit patterns travel widened to int32
    local = torch.from_numpy(y_local.astype(np.int32).reshape(-1))
    gathered = torch.empty(world * local.numel(), dtype=torch.int32)
    dist.all_gather_into_tensor(gathered, local)
    y = tp.unshard_host(gathered.numpy().astype(np.uint16), world, batch, shard.rows)
    if rank == 0:
        full = orc.gemv(sid, rows, cols, qt.padded_cols, qt.scales, qt.payload, x, batch)
        np.save(os.path.join(result_dir, "ok.npy"), np.array([np.array_equal(y, full)]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("sid,rows,cols,batch", [(7, 64, 200, 3), (4, 96, 256, 5)])
def test_tp_world2_gloo_matches_single_device(tmp_path, sid, rows, cols, batch):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, sid, rows, cols, batch, str(tmp_path)), nprocs=2, join=True)
    assert bool(np.load(tmp_path / "ok.npy")[0])


def test_shard_range_and_tensor():
    assert tp.shard_range(8192, 8, 3) == (3072, 1024)
    assert tp.shard_range(57344, 8, 7) == (50176, 7168)  # 70B gate_up, last rank
    with pytest.raises(ValueError):
        tp.shard_range(100, 3, 0)
    with pytest.raises(ValueError):
        tp.shard_range(64, 2, 2)
    from helpers import random_payload
    qt = random_payload(7, 64, 100, seed=2)
    parts = [tp.shard_tensor(qt, 4, r) for r in range(4)]
    assert np.array_equal(np.concatenate([p.payload for p in parts]), qt.payload)
    assert np.array_equal(np.concatenate([p.scales for p in parts]), qt.scales)
    assert all(p.padded_cols == qt.padded_cols and p.rows == 16 for p in parts)


def test_unshard_host_permutation():
    P, M, n = 3, 2, 4
    g = np.arange(P * M * n).reshape(P, M, n)
    y = tp.unshard_host(g, P, M, n)
    for p in range(P):
        assert np.array_equal(y[:, p * n:(p + 1) * n], g[p])


@pytest.mark.gpu
def test_tp_device_path_world1_and_unshard_kernel(cuda, orc):
    """World size 1 ShardedLinear == full linear; amsq_tp_unshard == unshard_host."""
    from helpers import check_linear, gaussian_x, quantized_gaussian
    from paper_2510_16045_b200._lib import check, lib
    sid, rows, cols, batch = 7, 512, 1000, 4
    qt = quantized_gaussian(sid, rows, cols, seed=3)
    x = gaussian_x(batch, cols, seed=4)
    xt = torch.from_numpy(x.view(np.float16).reshape(batch, cols)).to(cuda)
    y = tp.ShardedLinear(qt, device=0)(xt).cpu().numpy().view(np.uint16)
    yref = orc.gemv(sid, rows, cols, qt.padded_cols, qt.scales, qt.payload, x, batch)
    _, yabs = orc.gemv_f64(sid, rows, cols, qt.padded_cols, qt.scales, qt.payload, x, batch)
    check_linear(y, yref, yabs)
    # P shard outputs computed on one device, gathered by hand, un-sharded by the kernel
    P = 4
    outs = []
    for r in range(P):
        row0, n = tp.shard_range(rows, P, r)
        from paper_2510_16045_b200 import DeviceWeight
        outs.append(DeviceWeight(qt, device=0, row0=row0, nrows=n).linear(xt))
    gathered = torch.stack(outs).contiguous()  # [P][M][N/P]
    out = torch.empty(batch, rows, dtype=torch.float16, device=cuda)
    check(lib().amsq_tp_unshard(gathered.data_ptr(), P, batch, rows // P, out.data_ptr(),
                                torch.cuda.current_stream().cuda_stream), "unshard")
    want = tp.unshard_host(gathered.cpu().numpy(), P, batch, rows // P)
    assert np.array_equal(out.cpu().numpy(), want)
    check_linear(out.cpu().numpy().view(np.uint16), yref, yabs)


def _comm_init_all(ndev):
    import ctypes as C
    from paper_2510_16045_b200._lib import check, lib
    devs = (C.c_int * ndev)(*range(ndev))
    comms = (C.c_void_p * ndev)()
    check(lib().amsq_nccl_comm_init_all(ndev, devs, comms), "nccl_comm_init_all")
    return comms


@pytest.mark.gpu
@pytest.mark.parametrize("sid", [4, 7])
def test_tp_nccl_single_process_all_gpus(cuda, orc, sid):
    """one process, ncclCommInitAll over every visible GPU (1 on the
    single-GPU box, where the all-gather is a 1-rank NCCL collective), amsq_linear_tp_group:
    per-rank fused linear on its N-shard, grouped ncclAllGather, unshard. The gathered
    [M][N] output on every rank must meet the bar against the full reference gemv."""
    import ctypes as C
    from helpers import check_linear, gaussian_x, random_payload
    from paper_2510_16045_b200 import DeviceWeight
    from paper_2510_16045_b200._lib import check, lib
    P = torch.cuda.device_count()
    rows, cols, batch = 1024 * P, 8192, 4
    qt = random_payload(sid, rows, cols, seed=P)
    x = gaussian_x(batch, cols, seed=2)
    comms = _comm_init_all(P)
    shards, xs, ys, scr, streams = [], [], [], [], []
    need = 2 * batch * (rows // P) * (P + 1)
    for r in range(P):
        row0, n = tp.shard_range(rows, P, r)
        shards.append(DeviceWeight(qt, device=r, row0=row0, nrows=n))
        with torch.cuda.device(r):
            xs.append(torch.from_numpy(x.view(np.float16).reshape(batch, cols)).to(f"cuda:{r}"))
            ys.append(torch.empty(batch, rows, dtype=torch.float16, device=f"cuda:{r}"))
            scr.append(torch.empty(need, dtype=torch.uint8, device=f"cuda:{r}"))
            streams.append(torch.cuda.current_stream(r).cuda_stream)
    arr = lambda vals: (C.c_void_p * P)(*vals)  # noqa: E731
    check(lib().amsq_linear_tp_group(P, arr([s.handle for s in shards]),
                                     arr([t.data_ptr() for t in xs]), batch,
                                     arr([t.data_ptr() for t in ys]),
                                     arr([t.data_ptr() for t in scr]), need, comms,
                                     arr(streams)), "linear_tp_group")
    for r in range(P):
        torch.cuda.synchronize(r)
    yref = orc.gemv(sid, rows, cols, qt.padded_cols, qt.scales, qt.payload, x, batch)
    _, yabs = orc.gemv_f64(sid, rows, cols, qt.padded_cols, qt.scales, qt.payload, x, batch)
    for r in range(P):
        check_linear(ys[r].cpu().numpy().view(np.uint16), yref, yabs)
    for r in range(P):
        lib().amsq_nccl_comm_destroy(comms[r])


@pytest.mark.gpu
def test_tp_nccl_rank_comm_and_linear_tp(cuda, orc):
    """The per-process form the bench uses at N>1: amsq_nccl_unique_id +
    amsq_nccl_comm_init_rank, then amsq_linear_tp (here world 1: a 1-rank ncclAllGather)."""
    import ctypes as C
    from helpers import check_linear, gaussian_x, random_payload
    from paper_2510_16045_b200 import DeviceWeight
    from paper_2510_16045_b200._lib import check, lib
    uid = (C.c_uint8 * 128)()
    check(lib().amsq_nccl_unique_id(uid, 128), "unique_id")
    comm = C.c_void_p()
    check(lib().amsq_nccl_comm_init_rank(uid, 128, 1, 0, 0, C.byref(comm)), "init_rank")
    sid, rows, cols, batch = 7, 2048, 4096, 16
    qt = random_payload(sid, rows, cols, seed=9)
    x = gaussian_x(batch, cols, seed=1)
    dw = DeviceWeight(qt)
    xt = torch.from_numpy(x.view(np.float16).reshape(batch, cols)).to(cuda)
    y = torch.empty(batch, rows, dtype=torch.float16, device=cuda)
    need = 2 * batch * rows * 2
    scr = torch.empty(need, dtype=torch.uint8, device=cuda)
    check(lib().amsq_linear_tp(dw.handle, xt.data_ptr(), batch, y.data_ptr(), scr.data_ptr(),
                               need, comm, 1, torch.cuda.current_stream().cuda_stream), "tp")
    yref = orc.gemv(sid, rows, cols, qt.padded_cols, qt.scales, qt.payload, x, batch)
    _, yabs = orc.gemv_f64(sid, rows, cols, qt.padded_cols, qt.scales, qt.payload, x, batch)
    check_linear(y.cpu().numpy().view(np.uint16), yref, yabs)
    check(lib().amsq_nccl_comm_destroy(comm), "destroy")


@pytest.mark.gpu
@pytest.mark.parametrize("sid", [4, 7])
@pytest.mark.parametrize("P", [2, 4, 8])
def test_tp_fused_epilogue_matches_reference_and_nccl_path(cuda, orc, sid, P):
    """§8(f)2: amsq_linear_tp_fused -- each rank's K2 epilogue stores its [M][N/P] slice into
    EVERY rank's arena, then a flag barrier. With one GPU the P ranks are virtual (same
    device, one stream each, launched concurrently); with P GPUs they are real peers. Every
    rank must end with the identical full output, equal bit for bit to the per-shard K2
    outputs concatenated (the NCCL path) and within the bar of the reference gemv. Two calls
    at different arena offsets exercise the device-side epochs."""
    from helpers import check_linear, gaussian_x, random_payload
    from paper_2510_16045_b200 import DeviceWeight
    from paper_2510_16045_b200._lib import lib
    ndev = torch.cuda.device_count()
    devices = [r % ndev for r in range(P)]
    n_local, cols = 512, 4096
    rows = n_local * P
    qt = random_payload(sid, rows, cols, seed=P + sid)
    grp = tp.FusedTPGroup(devices, arena_bytes=2 * 2 * 40 * rows)
    try:
        shards = [DeviceWeight(qt, device=devices[r], row0=r * n_local, nrows=n_local)
                  for r in range(P)]
        streams = [torch.cuda.Stream(device=devices[r]) for r in range(P)]
        for call, batch in enumerate((1, 40)):
            x = gaussian_x(batch, cols, seed=batch)
            xs = [torch.from_numpy(x.view(np.float16).reshape(batch, cols)).to(f"cuda:{d}")
                  for d in devices]
            off = call * 2 * 40 * rows
            for r in range(P):
                streams[r].wait_stream(torch.cuda.current_stream(devices[r]))
                grp.linear(r, shards[r], xs[r], y_offset=off, stream=streams[r])
            for s in streams:
                s.synchronize()
            assert all(grp.error(r) == 0 for r in range(P))
            outs = [grp.arena(r)[off:off + 2 * batch * rows].view(torch.float16)
                    .reshape(batch, rows).cpu() for r in range(P)]
            for r in range(1, P):
                assert torch.equal(outs[r], outs[0]), f"rank {r} differs"
            # the fused epilogue is a K2 epilogue at every batch: compare with the per-shard
            # K2 outputs even where the dispatch would pick K3 (batch 40 >= the crossover)
            prev = lib().amsq_debug_set_k3_min_batch(100000)
            try:
                local = torch.cat([shards[r].linear(xs[r]).cpu() for r in range(P)], dim=1)
            finally:
                lib().amsq_debug_set_k3_min_batch(prev)
            assert torch.equal(outs[0], local)
            yref = orc.gemv(sid, rows, cols, qt.padded_cols, qt.scales, qt.payload, x, batch)
            _, yabs = orc.gemv_f64(sid, rows, cols, qt.padded_cols, qt.scales, qt.payload, x,
                                   batch)
            check_linear(outs[0].numpy().view(np.uint16), yref, yabs)
    finally:
        grp.close()
