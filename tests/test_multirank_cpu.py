"""Host logic of the row-sharded N > 1 path, world_size 2 over gloo on CPU (north star:
"Phi is sharded by rows: each GPU computes its partial g, and an NCCL all-reduce ...
sums the length-N g, after which thresholding is replicated").

Checked: shard_rows partition; per-shard codes equal the rows of the whole-matrix codes
(global Philox counters); the all-reduced max scale equals the global c (reading c3);
the all-reduced (sum) per-shard adjoints equal the whole adjoint; the replicated H_s is
then identical on every rank; and the NCCL unique id produced by libiht on rank 0
reaches every rank intact through torch.distributed.broadcast_object_list.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import iht as OI
        from oracle import quantize as OQ
        from paper_1802_04907_b200.problem import shard_rows
        from workloads import gen as G

        p = G.gaussian_problem(512, 700, 9, cfg_id=91, b_phi=4, K=2)
        rows, row0 = shard_rows(p.M, world, rank)
        phi_shard = p.phi[row0:row0 + rows]
        # global scale by all-reduce(max) of the shard maxima
        c_loc = torch.tensor([float(OQ.scale_c(phi_shard))], dtype=torch.float64)
        dist.all_reduce(c_loc, op=dist.ReduceOp.MAX)
        c = np.float32(c_loc.item())
        codes, _ = OQ.quantize_matrix(phi_shard, 4, 0, p.seed, 0, c=c, row_offset=row0)
        A = OQ.dequantize(codes, c, 4, 0)
        rng = np.random.default_rng(5)
        r_full = rng.standard_normal(p.M)
        g = torch.from_numpy(OI.adjoint(A, r_full[row0:row0 + rows]))
        dist.all_reduce(g, op=dist.ReduceOp.SUM)
        xi, xv = OI.hard_threshold(g.numpy(), p.s)
        # NCCL unique id from libiht (host API, no GPU needed) broadcast over gloo
        uid = None
        try:
            import ctypes
            from paper_1802_04907_b200 import _lib
            lib = _lib.load()
            buf = (ctypes.c_uint8 * 128)()
            rc = lib.iht_comm_unique_id(ctypes.cast(buf, ctypes.c_void_p)) if rank == 0 else 0
            obj = [bytes(buf) if rank == 0 else None, rc]
            dist.broadcast_object_list(obj, src=0)
            uid = (obj[0], obj[1])
        except Exception as e:  # noqa: BLE001
            uid = ("error", repr(e))
        out_q.put((rank, rows, row0, float(c), codes, g.numpy(), xi, xv, uid))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_row_sharded_host_logic_world2():
    from oracle import iht as OI
    from oracle import quantize as OQ
    from workloads import gen as G

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=240) for _ in range(world)], key=lambda t: t[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0

    p = G.gaussian_problem(512, 700, 9, cfg_id=91, b_phi=4, K=2)
    c = OQ.scale_c(p.phi)
    full_codes, _ = OQ.quantize_matrix(p.phi, 4, 0, p.seed, 0, c=c)
    g_full = OI.adjoint(OQ.dequantize(full_codes, c, 4, 0), np.random.default_rng(5).standard_normal(p.M))
    assert [r[1] for r in res] == [256, 256] and [r[2] for r in res] == [0, 256]
    for rank, rows, row0, cr, codes, g, xi, xv, uid in res:
        assert np.float32(cr) == c                                          # global c on every rank
        np.testing.assert_array_equal(codes, full_codes[:, row0:row0 + rows])  # global counters
        np.testing.assert_allclose(g, g_full, rtol=1e-12, atol=1e-12)       # sum of partial adjoints
    # replicated threshold is identical on both ranks
    assert res[0][6].tolist() == res[1][6].tolist()
    np.testing.assert_array_equal(res[0][7], res[1][7])
    # NCCL id: identical 128 bytes on both ranks (or NCCL unavailable on this host)
    u0, u1 = res[0][8], res[1][8]
    if u0[0] != "error" and u0[1] == 0:
        assert u0 == u1 and len(u0[0]) == 128 and any(u0[0])


def test_shard_rows_partition():
    from paper_1802_04907_b200.problem import shard_rows
    for world in (1, 2, 4, 8):
        spans = [shard_rows(65536, world, r) for r in range(world)]
        assert sum(s[0] for s in spans) == 65536
        assert [s[1] for s in spans] == [r * 65536 // world for r in range(world)]
        assert all(s[0] % 256 == 0 for s in spans)
    with pytest.raises(ValueError):
        shard_rows(1000, 3, 0)
