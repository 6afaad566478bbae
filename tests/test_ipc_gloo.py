"""Multi-process host logic of the one-process-per-GPU communicator, on CPU
with the gloo backend (world size 2): handle blobs are exchanged through
torch.distributed exactly as Communicator.ipc / bench.py do, and the gathered
set is validated by the library (flux_ipc_blobs_check) before any mapping."""
import ctypes as C
import os
import socket
import struct

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2406_06858_b200 import _native as N

MAGIC = 0xF1 << 24 | 0xB200


def blob(rank, tp, heap, magic=MAGIC):
    # IpcBlob: u32 magic; i32 rank, tp, device; u64 heap_bytes; i32 pid, pad; 64-byte cudaIpcMemHandle_t
    return struct.pack("<IiiiQii64s", magic, rank, tp, rank, heap, os.getpid(), 0, bytes([rank]) * 64)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    heap = 1 << 30
    mine = blob(rank, world, heap)
    out = [None] * world
    dist.all_gather_object(out, mine)
    joined = C.create_string_buffer(b"".join(out), len(mine) * world)
    rc_ok = N.lib().flux_ipc_blobs_check(joined, world, heap)
    rc_heap = N.lib().flux_ipc_blobs_check(joined, world, heap * 2)
    swapped = C.create_string_buffer(b"".join(reversed(out)), len(mine) * world)
    rc_order = N.lib().flux_ipc_blobs_check(swapped, world, heap)
    # max-over-ranks of per-rank step times, as bench.py reduces them
    import torch
    t = torch.tensor([10.0 + rank])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    results[rank] = (rc_ok, rc_heap, rc_order, [struct.unpack_from("<i", b, 4)[0] for b in out], t.item())
    dist.destroy_process_group()


def test_blob_size_matches_abi():
    assert N.lib().flux_comm_ipc_blob_bytes() == len(blob(0, 1, 1))


def test_blob_exchange_and_validation_world_size_2():
    ctx = mp.get_context("spawn")
    manager = ctx.Manager()
    results = manager.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, results)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for r in range(2):
        ok, bad_heap, bad_order, ranks, tmax = results[r]
        assert ok == N.OK
        assert bad_heap == N.ERR_CONFIG          # heaps must be symmetric
        assert bad_order == N.ERR_DIRECTORY      # blob r must carry rank r
        assert ranks == [0, 1]
        assert tmax == 11.0


def test_blob_check_rejects_bad_magic_and_tp():
    good = [blob(r, 2, 4096) for r in range(2)]
    bad = C.create_string_buffer(blob(0, 2, 4096, magic=0) + good[1], 2 * len(good[0]))
    assert N.lib().flux_ipc_blobs_check(bad, 2, 4096) == N.ERR_DIRECTORY
    wrong_tp = C.create_string_buffer(blob(0, 4, 4096) + blob(1, 4, 4096), 2 * len(good[0]))
    assert N.lib().flux_ipc_blobs_check(wrong_tp, 2, 4096) == N.ERR_CONFIG
    msg = N.lib().flux_last_error().decode()
    assert "tp=4" in msg
