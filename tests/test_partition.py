"""Batch partitioner (a10) -- host logic, plus a world_size-2 gloo run of the
gather path (the same code the multi-GPU bench uses, over CPU tensors)."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

from paper_1710_04985_b200 import partition


@pytest.mark.parametrize("total,ws", [(64, 1), (64, 2), (64, 4), (64, 8), (10, 3), (3, 8), (0, 4)])
def test_block_range_covers_exactly(total, ws):
    ranges = partition.all_ranges(total, ws)
    assert ranges[0][0] == 0 and ranges[-1][1] == total
    for (a, b), (c, d) in zip(ranges, ranges[1:]):
        assert b == c and a <= b
    sizes = [b - a for a, b in ranges]
    assert max(sizes) - min(sizes) <= 1


def test_block_range_rejects_bad_args():
    with pytest.raises(ValueError):
        partition.block_range(8, 0, 0)
    with pytest.raises(ValueError):
        partition.block_range(8, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, total, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    a, b = partition.block_range(total, ws, rank)
    n = 5
    # each rank "solves" its columns: column r of the result is r + 100*i
    local = torch.tensor([[float(r + 100 * i) for r in range(a, b)] for i in range(n)],
                         dtype=torch.float64).reshape(n, b - a)
    full = partition.gather_columns(local, total)
    out[rank] = full.tolist()
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [64, 7])
def test_gather_columns_gloo_world2(total):
    ws = 2
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(ws, port, total, out), nprocs=ws, join=True)
    expect = [[float(r + 100 * i) for r in range(total)] for i in range(5)]
    for r in range(ws):
        assert out[r] == expect


def test_break_even_solves_matches_brute_force():
    """bench.break_even_solves = Table 7's n_s: the smallest n >= 1
    with setup_a + n solve_a < setup_b + n solve_b, checked by scanning n."""
    import importlib.util
    import os
    import random
    spec = importlib.util.spec_from_file_location("bench", os.path.join(os.path.dirname(os.path.dirname(
        os.path.abspath(__file__))), "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    rng = random.Random(3)
    for _ in range(400):
        sa, sb = rng.uniform(0, 0.2), rng.uniform(0, 0.2)
        ta, tb = rng.uniform(1e-5, 3e-3), rng.uniform(1e-5, 3e-3)
        got = bench.break_even_solves(sa, ta, sb, tb)
        want = None
        for n in range(1, 200000):
            if sa + n * ta < sb + n * tb:
                want = n
                break
        if want is None:
            assert got is None or got >= 200000, (sa, ta, sb, tb, got)
        else:
            assert got == want, (sa, ta, sb, tb, got, want)


@pytest.mark.parametrize("ws", [1, 2, 3, 4, 8])
def test_factor_assignment_covers_and_balances(ws):
    import random
    rng = random.Random(ws)
    for _ in range(50):
        w = [rng.randint(1, 1000) for _ in range(rng.randint(0, 40))]
        own = partition.factor_assignment(w, ws)
        assert len(own) == ws
        flat = sorted(i for o in own for i in o)
        assert flat == list(range(len(w)))                 # each factor exactly once
        loads = [sum(w[i] for i in o) for o in own]
        if w:
            assert max(loads) <= sum(w) / ws + max(w)       # LPT bound
        assert own == partition.factor_assignment(w, ws)    # deterministic


def test_block_jacobi_workload_is_block_diagonal_ilu():
    import numpy as np
    import workloads
    t = workloads.slab_thicknesses(32, 5, seed=6)
    assert sum(t) == 32 and min(t) >= 1 and len(t) == 5
    blocks = workloads.block_jacobi_ilu0((6, 5, 32), 27, 5, seed=6)
    assert [b.n for b in blocks] == [6 * 5 * tz for tz in t]
    # each block is the ILU(0) of its own slab's stencil: same pattern as the slab matrix
    for b, tz in zip(blocks, t):
        a = workloads.stencil((6, 5, tz), 27, "full")
        assert np.array_equal(b.rowptr, a.rowptr) and np.array_equal(b.colidx, a.colidx)
