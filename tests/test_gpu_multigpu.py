"""Two-GPU runs of libiht's sharded solvers (§8(e)), one process per GPU over NCCL, each
compared with the float64 oracle's trajectory (Algorithm 1):

* row shards (single observation): every rank quantises rows [p M/P, (p+1) M/P) of each
  copy; per iteration the partial g are reduce-scattered, each rank selects its column
  slice, the candidate lists are all-gathered and merged;
* column shards (batched observations, tcgen05 path): the forward partials are all-reduced,
  the adjoint is local, the per-rank top-s candidates are all-gathered and merged.

The summation order of the exchanged sums differs from one GPU's, so the bar is the oracle's
(identical supports up to its first near-tie, x within 1e-4 / 1e-3 relative l2), and both
ranks must hold bit-identical replicated iterates.  Skipped on a box with fewer than two
GPUs (the round-end box has one: this path's host logic is covered by
tests/test_multirank_cpu.py over gloo)."""
import os
import socket

import numpy as np
import pytest
import torch

from oracle import iht as OI
from workloads import gen as G

from helpers import check_trajectory, near_tie

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                                 reason="needs two GPUs")]
WORLD = 2


def _row_problem():
    return G.gaussian_problem(1024, 4096, 20, cfg_id=41, b_phi=4, n_iter=20, mu=0.5, K=4)


def _col_problem():
    return G.radio_problem(cfg_id=42, A=12, grid=64, n_src=6, n_iter=12, K=4, batch=4)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, port, kind, q):
    import torch.distributed as dist
    from paper_1802_04907_b200 import iht
    from paper_1802_04907_b200.problem import build_pool
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(WORLD))
    torch.cuda.set_device(rank)
    dev = torch.device(f"cuda:{rank}")
    dist.init_process_group("nccl", rank=rank, world_size=WORLD)
    try:
        if kind == "rows":
            p = _row_problem()
            pool, _, _, rows, row0 = build_pool(p, rank, WORLD, dev, True)
            y = torch.from_numpy(np.ascontiguousarray(p.y[row0:row0 + rows])).to(dev)
            nrhs = 1
        else:
            p = _col_problem()
            pool, _, _, _, _ = build_pool(p, rank, WORLD, dev, True, shard="cols")
            nrhs = p.meta["batch_y"].shape[1]
            y = torch.from_numpy(np.ascontiguousarray(p.meta["batch_y"].T)).to(dev)
        comm = iht.Comm(rank, WORLD, rank)
        sol = iht.Solver(pool, p.s, p.n_iter, p.mu, p.b_y, p.seed, comm=comm, trace=True, nrhs=nrhs)
        sol.run(y)
        torch.cuda.synchronize(dev)
        idx, val, nnz = (np.asarray(t) for t in sol.trace_arrays())
        sol.close()
        comm.close()
        q.put((rank, idx, val, nnz, None))
    except Exception as e:          # reported to the parent, which fails the test
        q.put((rank, None, None, None, repr(e)))
    finally:
        dist.destroy_process_group()


def _run(kind):
    ctx = torch.multiprocessing.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, kind, q)) for r in range(WORLD)]
    for pr in procs:
        pr.start()
    out = {}
    for _ in range(WORLD):
        rank, idx, val, nnz, err = q.get(timeout=600)
        assert err is None, f"rank {rank}: {err}"
        out[rank] = (idx, val, nnz)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for a, b in zip(out[0], out[1]):            # the replicated iterate: identical bits on both ranks
        assert np.array_equal(a, b)
    return out[0]


def test_two_gpu_row_sharded_solver_matches_oracle():
    p = _row_problem()
    idx, val, nnz = _run("rows")
    ref = OI.qniht(p.phi, p.y, p.s, p.n_iter, p.mu, p.b_phi, p.b_y, p.seed, p.K, record=True)
    checked = check_trajectory(ref.trace, idx, val, nnz, p.s, 1e-4)
    assert checked >= min(10, p.n_iter)


def test_two_gpu_column_sharded_batched_solver_matches_oracle():
    p = _col_problem()
    idx, val, nnz = _run("cols")
    Y = p.meta["batch_y"].T
    total = 0
    for b in range(Y.shape[0]):
        ref = OI.qniht(p.phi, Y[b], p.s, p.n_iter, p.mu, p.b_phi, p.b_y, p.seed, p.K, record=True, snapshot=b)
        for n, rec in enumerate(ref.trace):
            if near_tie(rec.a, rec.margin, p.s, rel=1e-3):
                break
            k = int(nnz[n, b])
            assert idx[n, b, :k].tolist() == rec.x_idx.tolist(), (b, n)
            err = np.linalg.norm(val[n, b, :k] - rec.x_val) / max(np.linalg.norm(rec.x_val), 1e-30)
            assert err <= 1e-3, (b, n, err)
            total += 1
    assert total >= Y.shape[0] * p.n_iter // 2
