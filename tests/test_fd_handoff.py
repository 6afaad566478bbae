"""The file-descriptor hand-off the NVLS setup of the one-process-per-GPU
communicator uses (rank 0's multicast handle is a POSIX fd): an abstract Unix
socket with SCM_RIGHTS, checked between real processes on the CPU."""
import multiprocessing as mp
import os
import tempfile

from paper_2406_06858_b200.comm import fd_receive, fd_server


def _client(name, q):
    fd = fd_receive(name, timeout_s=30.0)
    os.lseek(fd, 0, os.SEEK_SET)
    q.put(os.read(fd, 64))
    os.close(fd)


def test_fd_reaches_every_peer_process():
    with tempfile.TemporaryFile() as f:
        f.write(b"multicast handle stand-in")
        f.flush()
        fd = os.dup(f.fileno())
        name = "flux-nvls-test-%d" % os.getpid()
        server = fd_server(name, fd)
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        procs = [ctx.Process(target=_client, args=(name, q)) for _ in range(3)]
        for p in procs:
            p.start()
        server.serve(3, timeout_s=60.0)
        got = [q.get(timeout=60) for _ in procs]
        for p in procs:
            p.join(timeout=60)
            assert p.exitcode == 0
        assert got == [b"multicast handle stand-in"] * 3
        try:  # the server closed its copy of the fd
            os.fstat(fd)
            still_open = True
        except OSError:
            still_open = False
        assert not still_open
