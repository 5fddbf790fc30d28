"""The N > 1 bench path (replicas) on CPU with the gloo backend, world size 2:
the max-over-ranks device time and the whole-job throughput formula."""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, ws, port, q):
    import sys
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    t_local = [3.0, 5.0][rank]  # ms: rank 1 is the slowest replica
    t = bench.max_over_ranks(t_local, ws)
    bench.barrier(ws)
    q.put((rank, t, bench.replica_value(1e9, 10, t, ws)))
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_replicas_take_the_slowest_rank_and_sum_the_work():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=100) for _ in ps)
    for p in ps:
        p.join(timeout=30)
    assert [o[1] for o in out] == [5.0, 5.0]
    # 2 replicas x 10 steps x 1 GB in 5 ms -> 4000 GB/s
    assert all(abs(o[2] - 4000.0) < 1e-9 for o in out)


def test_bench_accounting_is_consistent():
    """The per-kernel algorithmic bytes add up to B_model (1344 N + 96 (nx+1)(ny+1)(nz+1));
    the K-C flop count is 6 FFTs of 5 L log2 L plus 72 flops per kz, per pencil of the padded xy grid."""
    import math
    import bench
    for n in [(256, 256, 128), (128, 128, 64), (8, 8, 8)]:
        assert sum(bench.kernel_bytes(*n).values()) == bench.b_model(*n)
        L = 2 * n[2]
        assert bench.kc_flops(*n) == 4 * n[0] * n[1] * (30 * L * math.log2(L) + 72 * L)
    assert abs(bench.FP64_NOMINAL_TFLOPS - 37.22496) < 1e-9
