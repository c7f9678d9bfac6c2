"""Host logic of the row-sharded N > 1 path, world_size 2 over gloo on CPU (north star:
"Phi is sharded by rows: each GPU computes its partial g, and an NCCL all-reduce ...
sums the length-N g, after which thresholding is replicated").

Checked: shard_rows partition; per-shard codes equal the rows of the whole-matrix codes
(global Philox counters); the all-reduced max scale equals the global c (reading c3);
the all-reduced (sum) per-shard adjoints equal the whole adjoint; the replicated H_s is
then identical on every rank; and the NCCL unique id produced by libiht on rank 0
reaches every rank intact through torch.distributed.broadcast_object_list.

Column-sharded batched path (config 5): shard_cols partition; shard codes
equal the whole-matrix columns (global Philox column quads); summed forward partials equal
the whole forward; local adjoints concatenate to the whole adjoint; the merge of the
all-gathered local top-s lists equals the global H_s (also on random tie-heavy inputs).
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


# ---------------------------------------------------------------------------------------
# Column-sharded batched path (config 5 at P > 1): each rank owns N/P pixels;
# forward partials are all-reduced (sum) into r, the local adjoint gives the local g, the
# local H_s candidates (global indices) are all-gathered and merged.  The merge of local
# top-s lists equals the global H_s with the same tie rule.
def _merge_topk(cands, s):
    """H_s of the union of candidate lists (idx increasing within and across lists)."""
    from oracle import iht as OI
    idx = np.concatenate([c[0] for c in cands]).astype(np.int64)
    val = np.concatenate([c[1] for c in cands])
    keep_pos, keep_val = OI.hard_threshold(val, s)     # positions in the concatenation (index order)
    return idx[keep_pos], keep_val


def _col_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import iht as OI
        from oracle import quantize as OQ
        from paper_1802_04907_b200.problem import shard_cols
        from workloads import gen as G

        p = G.radio_problem(cfg_id=92, A=10, grid=32, n_src=6, n_iter=3, K=2, batch=3)
        cols, col0 = shard_cols(p.N, world, rank)
        phi_shard = np.ascontiguousarray(p.phi[:, col0:col0 + cols])
        c_loc = torch.tensor([float(OQ.scale_c(phi_shard))], dtype=torch.float64)
        dist.all_reduce(c_loc, op=dist.ReduceOp.MAX)
        c = np.float32(c_loc.item())
        codes, _ = OQ.quantize_matrix(phi_shard, p.b_phi, 0, p.seed, 0, c=c, col_offset=col0)
        A = OQ.dequantize(codes, c, p.b_phi, 0)
        rng = np.random.default_rng(8)
        out = []
        for b in range(3):
            xi = np.sort(rng.choice(p.N, p.s, replace=False))
            xv = rng.standard_normal(p.s)
            yhat = p.meta["batch_y"][:, b].astype(np.complex128)
            mine = (xi >= col0) & (xi < col0 + cols)
            part = OI.forward(A, xi[mine] - col0, xv[mine], yhat if rank == 0 else np.zeros_like(yhat))
            rr = torch.from_numpy(np.stack([part.real, part.imag]))
            dist.all_reduce(rr, op=dist.ReduceOp.SUM)
            r = rr[0].numpy() + 1j * rr[1].numpy()
            g = OI.adjoint(A, r)
            a = g * 0.5
            a[xi[mine] - col0] += xv[mine]
            li, lv = OI.hard_threshold(a, p.s)
            gathered = [None] * world
            dist.all_gather_object(gathered, (li + col0, lv))
            out.append((r, g, _merge_topk(gathered, p.s), xi, xv))
        out_q.put((rank, cols, col0, float(c), codes, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_column_sharded_batched_host_logic_world2():
    from oracle import iht as OI
    from oracle import quantize as OQ
    from workloads import gen as G

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_col_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=240) for _ in range(world)], key=lambda t: t[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p = G.radio_problem(cfg_id=92, A=10, grid=32, n_src=6, n_iter=3, K=2, batch=3)
    c = OQ.scale_c(p.phi)
    full_codes, _ = OQ.quantize_matrix(p.phi, p.b_phi, 0, p.seed, 0, c=c)
    A = OQ.dequantize(full_codes, c, p.b_phi, 0)
    assert [r[1] for r in res] == [512, 512] and [r[2] for r in res] == [0, 512]
    for rank, cols, col0, cr, codes, out in res:
        assert np.float32(cr) == c
        np.testing.assert_array_equal(codes, full_codes[:, :, col0:col0 + cols])    # global Philox columns
    for b in range(3):
        r0, _, (mi0, mv0), xi, xv = res[0][5][b]
        r1, _, (mi1, mv1), _, _ = res[1][5][b]
        r_full = OI.forward(A, xi, xv, p.meta["batch_y"][:, b].astype(np.complex128))
        np.testing.assert_allclose(r0, r_full, rtol=1e-10, atol=1e-10)        # summed partial forwards
        np.testing.assert_array_equal(r0, r1)                                  # replicated after the sum
        g_full = OI.adjoint(A, r0)
        np.testing.assert_allclose(np.concatenate([res[0][5][b][1], res[1][5][b][1]]), g_full, rtol=1e-10,
                                   atol=1e-10)
        a = g_full * 0.5
        a[xi] += xv
        gi, gv = OI.hard_threshold(a, p.s)
        assert mi0.tolist() == gi.tolist() and mi1.tolist() == gi.tolist()    # merge == global H_s
        np.testing.assert_allclose(mv0, gv, rtol=0, atol=1e-12)


def test_merge_of_local_topk_equals_global_with_ties():
    from oracle import iht as OI
    rng = np.random.default_rng(3)
    for trial in range(50):
        N = int(rng.integers(20, 300))
        s = int(rng.integers(1, 25))
        a = np.round(rng.standard_normal(N), 1)          # many exact ties
        a[rng.random(N) < 0.2] = 0.0
        cuts = np.sort(rng.choice(np.arange(1, N), size=int(rng.integers(0, 5)), replace=False))
        bounds = [0, *cuts.tolist(), N]
        cands = []
        for lo, hi in zip(bounds[:-1], bounds[1:]):
            li, lv = OI.hard_threshold(a[lo:hi], s)
            cands.append((li + lo, lv))
        mi, mv = _merge_topk(cands, s)
        gi, gv = OI.hard_threshold(a, s)
        assert mi.tolist() == gi.tolist()
        np.testing.assert_array_equal(mv, gv)


def test_shard_cols_partition():
    from paper_1802_04907_b200.problem import shard_cols
    for world in (1, 2, 4, 8):
        spans = [shard_cols(65536, world, r) for r in range(world)]
        assert sum(s[0] for s in spans) == 65536 and all(s[1] % 16 == 0 for s in spans)
    with pytest.raises(ValueError):
        shard_cols(1000, 3, 0)


# ---------------------------------------------------------------------------------------
# Row-sharded single-observation path with the SHARDED select (libiht's iht_solver at P > 1,
# fixed step): every rank holds the partial adjoint g_p of its rows over all N columns;
# g is reduce-scattered (rank p receives the summed columns [p N/P, (p+1) N/P)); each rank
# forms a = x + mu g on its columns and keeps their local top-s (global indices); the P lists
# are all-gathered and merged.  The merge equals the global H_s(x + mu sum_p g_p) on every rank.
def _rs_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import iht as OI
        from oracle import quantize as OQ
        from paper_1802_04907_b200.problem import shard_rows
        from workloads import gen as G

        p = G.gaussian_problem(512, 704, 24, cfg_id=93, b_phi=2, K=2)
        rows, row0 = shard_rows(p.M, world, rank)
        phi_shard = p.phi[row0:row0 + rows]
        c_loc = torch.tensor([float(OQ.scale_c(phi_shard))], dtype=torch.float64)
        dist.all_reduce(c_loc, op=dist.ReduceOp.MAX)
        c = np.float32(c_loc.item())
        A = OQ.dequantize(OQ.quantize_matrix(phi_shard, p.b_phi, 0, p.seed, 0, c=c, row_offset=row0)[0], c,
                          p.b_phi, 0)
        rng = np.random.default_rng(12)
        out = []
        for trial in range(3):
            xi = np.sort(rng.choice(p.N, p.s, replace=False))
            xv = rng.standard_normal(p.s)
            r_full = rng.standard_normal(p.M)
            g_part = torch.from_numpy(OI.adjoint(A, r_full[row0:row0 + rows]))
            nloc = p.N // world
            col0 = rank * nloc
            g_loc = torch.empty(nloc, dtype=torch.float64)
            try:
                dist.reduce_scatter_tensor(g_loc, g_part, op=dist.ReduceOp.SUM)
            except (RuntimeError, NotImplementedError, ValueError):
                # gloo without reduce-scatter: the same sums through an all-reduce, sliced
                t = g_part.clone()
                dist.all_reduce(t, op=dist.ReduceOp.SUM)
                g_loc = t[col0:col0 + nloc].clone()
            a = 0.7 * g_loc.numpy()
            mine = (xi >= col0) & (xi < col0 + nloc)
            a[xi[mine] - col0] += xv[mine]
            li, lv = OI.hard_threshold(a, p.s)
            gathered = [None] * world
            dist.all_gather_object(gathered, (li + col0, lv))
            out.append((xi, xv, r_full, _merge_topk(gathered, p.s)))
        out_q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_row_sharded_sharded_select_world2():
    from oracle import iht as OI
    from oracle import quantize as OQ
    from workloads import gen as G

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rs_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=240) for _ in range(world)], key=lambda t: t[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p = G.gaussian_problem(512, 704, 24, cfg_id=93, b_phi=2, K=2)
    c = OQ.scale_c(p.phi)
    A = OQ.dequantize(OQ.quantize_matrix(p.phi, p.b_phi, 0, p.seed, 0, c=c)[0], c, p.b_phi, 0)
    for t in range(3):
        xi, xv, r_full, (mi0, mv0) = res[0][1][t]
        mi1, mv1 = res[1][1][t][3]
        a = 0.7 * OI.adjoint(A, r_full)
        a[xi] += xv
        gi, gv = OI.hard_threshold(a, p.s)
        assert mi0.tolist() == gi.tolist() and mi1.tolist() == gi.tolist()     # merge == global H_s
        np.testing.assert_allclose(mv0, gv, rtol=1e-12, atol=1e-12)
        np.testing.assert_array_equal(mv0, mv1)                                 # replicated x


def test_bench_relaunch_command():
    """bench.py --gpus N without a launcher re-executes itself under torchrun, one rank per
    GPU on one node, rendezvous on 127.0.0.1."""
    import importlib.util
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(root, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    cmd = bench.relaunch_cmd(8, ["--gpus", "8", "--steps", "5"], 29555)
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=8" in cmd and "--master-addr=127.0.0.1" in cmd and "--master-port=29555" in cmd
    assert cmd[-4:] == ["--gpus", "8", "--steps", "5"] and cmd[-5].endswith("bench.py")


@pytest.mark.timeout(300)
def test_bench_launcher_dry_run_world2():
    """End to end on CPU: `python bench.py --gpus 2 --dry-run` starts two ranks under torchrun,
    they rendezvous (gloo), reduce over ranks, and rank 0 prints one JSON line."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, timeout=240, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["ranks_max"] == 1
    assert lines[0]["master"] == "127.0.0.1"
