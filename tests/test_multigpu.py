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


def _sweep_worker(rank, ws, port, q):
    import sys
    import numpy as np
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    units = bench.sweep_units((0, 1, 2), (1e5, 4e5))
    merged, mine = bench.distributed_sweep(units, _oracle_unit, rank, ws)
    q.put((rank, mine, {k: v.tolist() for k, v in merged.items()}))
    dist.destroy_process_group()


def _oracle_unit(unit):
    """One (frequency, station) system of a tiny layered sweep, solved by the oracle (dense LU of
    the c4-recipe 8^3 mini with the physical table, E0 of the station's triaxial transmitter) ->
    the 9 receiver couplings per source dipole by reciprocity."""
    import numpy as np
    from ie_workloads import make_config, layered_inputs as li, tool_frame
    from oracle import layered as lay
    f, s = unit
    cfg = make_config("c4lmini")
    med = li.medium(cfg, f)
    F = tool_frame(70.0, 45.0)
    tx = (0.05 + 0.1 * s) * F[2]
    srcs = [(tx, F[i]) for i in range(3)]
    rx = [tx + 0.6 * F[2]]
    T = li.table(cfg, med)
    sbz = lay.background_per_layer(cfg.n, cfg.origin, cfg.hvec, *cfg.background())
    ds = lay.contrast_layered(cfg.sigma(), sbz)
    E0 = li.incident(cfg, med, srcs)
    e0rx, h0 = li.receiver_inputs(cfg, med, srcs, rx)
    A = lay.dense_matrix_layered(T, ds)
    out = []
    for i in range(3):
        E = np.linalg.solve(A, E0[i].ravel()).reshape(E0[i].shape)
        out.append([lay.receiver_coupling(E, ds, e0rx[d], h0[i, d], cfg.h ** 3, med.omega) for d in range(len(e0rx))])
    return np.array(out)


@pytest.mark.timeout(300)
def test_distributed_sweep_solves_each_unit_once_and_merges_like_one_rank():
    """World size 2 (gloo): the (frequency, station) systems of a sweep are split between the
    ranks, every unit is solved exactly once, and the merged receiver couplings equal the
    single-rank run."""
    import sys
    import numpy as np
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_sweep_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=250) for _ in ps)
    for p in ps:
        p.join(timeout=30)
    units = bench.sweep_units((0, 1, 2), (1e5, 4e5))
    mine = [tuple(u) for o in out for u in o[1]]
    assert sorted(mine) == sorted(units) and len(mine) == len(set(mine))  # each unit exactly once
    assert out[0][2].keys() == out[1][2].keys() == set(units)
    single, _ = bench.distributed_sweep(units, _oracle_unit, 0, 1)
    for u in units:
        assert np.array_equal(np.array(out[0][2][u]), single[u])
        assert np.array_equal(np.array(out[1][2][u]), single[u])


def _table_worker(rank, ws, port, q):
    import sys
    import numpy as np
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    from ie_workloads import make_config, layered_inputs as li
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    cfg = make_config("c3lmini")
    T = bench.shared_table(cfg, li.medium(cfg), rank, ws)
    q.put((rank, T))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_shared_table_is_generated_once_and_broadcast():
    """N > 1 ranks: rank 0 generates the layered table, the others receive it by broadcast --
    identical bytes on every rank, equal to a local generation."""
    import sys
    import numpy as np
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from ie_workloads import make_config, layered_inputs as li
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_table_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=250) for _ in ps)
    for p in ps:
        p.join(timeout=30)
    cfg = make_config("c3lmini")
    ref = li.table(cfg, li.medium(cfg))
    assert np.array_equal(out[0], ref) and np.array_equal(out[1], ref)
