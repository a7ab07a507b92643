"""Multi-process paths with real per-rank solves (gloo process group, every
rank on cuda:0): the batch partitioners of §8(e) -- RHS columns (a10) and
independent factors (NEXT-4) -- each rank solving only what it owns, results
gathered and compared bit for bit with one process solving everything."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _factor_worker(rank, ws, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    torch.cuda.set_device(0)
    import workloads
    from paper_1710_04985_b200 import partition
    from paper_1710_04985_b200 import sptrsv as S
    blocks, p = workloads.config(6, scale=0.25)
    owned = partition.factor_assignment([int(b.rowptr[-1]) for b in blocks], ws)[rank]
    res = {}
    for i in owned:
        b = blocks[i]
        hl = S.from_csr(b, "lower", "unit", algo="auto")
        hu = S.from_csr(b, "upper", "non_unit", algo="auto")
        rhs = torch.from_numpy(workloads.rhs(b.n, 1, seed=p["seed"] + i)[:, 0]).cuda()
        res[i] = hu.solve(hl.solve(rhs)).cpu().numpy().tolist()
        assert hl.solve_status() == "SUCCESS" and hu.solve_status() == "SUCCESS"
    gathered = [None] * ws
    dist.all_gather_object(gathered, res)
    if rank == 0:
        merged = {}
        for g in gathered:
            merged.update(g)
        out["x"] = merged
        out["owned"] = [partition.factor_assignment([int(b.rowptr[-1]) for b in blocks], ws)[r] for r in range(ws)]
    dist.destroy_process_group()


def _rhs_worker(rank, ws, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    torch.cuda.set_device(0)
    import workloads
    from paper_1710_04985_b200 import partition
    from paper_1710_04985_b200 import sptrsv as S
    m, _ = workloads.config(5, scale=0.25)
    a, e = partition.block_range(64, ws, rank)
    b = torch.from_numpy(workloads.rhs_columns(m.n, range(a, e))).cuda()
    x = S.from_csr(m, algo="auto").solve(b).cpu()
    full = partition.gather_columns(x, 64)
    if rank == 0:
        out["x"] = full.numpy()
    dist.destroy_process_group()


def test_factor_batch_two_ranks_equal_one_process():
    import workloads
    from paper_1710_04985_b200 import sptrsv as S
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_factor_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    owned = out["owned"]
    assert sorted(owned[0] + owned[1]) == list(range(16)) and owned[0] and owned[1]
    blocks, p = workloads.config(6, scale=0.25)
    for i, b in enumerate(blocks):
        hl = S.from_csr(b, "lower", "unit", algo="auto")
        hu = S.from_csr(b, "upper", "non_unit", algo="auto")
        rhs = torch.from_numpy(workloads.rhs(b.n, 1, seed=p["seed"] + i)[:, 0]).cuda()
        x1 = hu.solve(hl.solve(rhs)).cpu().numpy()
        assert np.array_equal(np.asarray(out["x"][i]), x1), i


def test_rhs_partition_two_ranks_equal_one_process():
    import workloads
    from paper_1710_04985_b200 import sptrsv as S
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_rhs_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    m, _ = workloads.config(5, scale=0.25)
    b = torch.from_numpy(workloads.rhs_columns(m.n, range(64))).cuda()
    x1 = S.from_csr(m, algo="auto").solve(b).cpu().numpy()
    assert np.array_equal(out["x"], x1)
