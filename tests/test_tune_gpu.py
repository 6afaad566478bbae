"""The autotuner's device objective and correctness gate on a real B200
(SURVEY §8f row 3): every config of the reference knob space (plus CTA group
and AG transfer engine) runs, passes the cuBLAS-sampled gate, and the cache
serves the winner on the second call."""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2406_06858_b200 as fx  # noqa: E402
from paper_2406_06858_b200 import _native as N  # noqa: E402
from paper_2406_06858_b200 import tune as T  # noqa: E402


def _comm_with_inputs(p, seed):
    comm = fx.Communicator(p.tp, [0] * p.tp, heap_bytes=fx.required_heap_bytes(p))
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    for r in range(p.tp):
        for kind in (N.BUF_A_SHARD, N.BUF_B_SHARD):
            t = comm.tensor(r, kind, p)
            t.copy_((torch.rand(t.shape, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16))
    torch.cuda.synchronize()
    return comm


@pytest.mark.parametrize("pattern", [fx.ALLGATHER_GEMM, fx.GEMM_REDUCESCATTER])
def test_tuner_on_device(pattern, tmp_path):
    p = fx.ProblemSpec(1024, 1024, 512, 4, pattern)
    comm = _comm_with_inputs(p, 3 + pattern)
    try:
        ks = T.default_knob_space(p)
        ks.gemm_tile_shapes = [fx.TileShape(128, 128), fx.TileShape(64, 128)]
        cache = str(tmp_path / "cache.json")
        args = dict(measure=T.gpu_measure(comm, p, 3), verify=T.gpu_verify(comm, p), repetitions=3,
                    cache_path=cache, machine=T.machine_id())
        res = T.tune(p, ks, **args)
        assert len(res.table) == len(T.enumerate_knobs(p, ks))
        assert all(e.objective_us > 0 for e in res.table)
        assert res.objective_us == min(e.objective_us for e in res.table)
        again = T.tune(p, ks, **args)
        assert again.from_cache and again.best_config == res.best_config
    finally:
        comm.close()


def test_tuner_gate_catches_a_wrong_result():
    p = fx.ProblemSpec(512, 512, 256, 2, fx.ALLGATHER_GEMM)
    comm = _comm_with_inputs(p, 9)
    try:
        verify = T.gpu_verify(comm, p)
        cfg = T.enumerate_knobs(p, T.default_knob_space(p))[0]
        verify(cfg)  # a correct run passes
        # Corrupt one rank's weights after the reference was taken: the gate must fire.
        comm.tensor(1, N.BUF_B_SHARD, p).mul_(2)
        with pytest.raises(AssertionError):
            verify(cfg)
    finally:
        comm.close()
