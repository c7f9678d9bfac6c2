"""Set up a problem's quantised pool on the device (one-time per operator; not timed).

Generates (config 4: on the device, block-wise, never resident) and quantises this
rank's row shard of Phi into the pool of K copies, with the global scale c all-reduced
across ranks (reading c3).  Used by bench.py and by the full-size parity tests, so the
tests exercise exactly the configuration the bench times.
"""
import time

import numpy as np


def shard_rows(M, world, rank):
    """Row shard of rank `rank` (north star: Phi sharded by rows).  Requires M % world == 0
    and shards that are whole 256-row blocks (so the block-wise quantiser can write them)."""
    if M % world:
        raise ValueError("row sharding needs M divisible by the GPU count")
    rows = M // world
    return rows, rank * rows


def shard_cols(N, world, rank):
    """Column shard of rank `rank` (batched path): equal widths, multiples of 16
    (the tiled code layout and the quantiser's Philox column quads)."""
    if N % (16 * world):
        raise ValueError("column sharding needs N divisible by 16 x the GPU count")
    cols = N // world
    return cols, rank * cols


def _timed(fn):
    """Run fn() between two CUDA events on the current stream; returns the event pair."""
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    return e0, e1


def _quantize_stats(t, qev, components, K, bits):
    """Quantiser throughput ((4 + K b / 8) bytes per real component for one fp32
    read emitting K copies) from the event-timed launches."""
    import torch
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in qev)
    t["quantize_ms"] = ms
    t["quantize_launches"] = len(qev)
    t["quantize_bytes"] = int(components * 4 + K * components * bits // 8)
    t["quantize_GBps"] = t["quantize_bytes"] / (ms / 1e3) / 1e9 if ms > 0 else None


def build_pool(p, rank, world, dev, dist_on, shard="rows"):
    """Generate (config 4: on the device, block-wise) and quantise this rank's shard of Phi
    (row shard, or column shard for the batched path) into the pool of K copies.
    Returns (pool, c_phi, preprocess timings, rows, row0)."""
    import torch
    from . import iht
    if shard == "cols":
        return _build_pool_cols(p, rank, world, dev, dist_on)
    rows, row0 = shard_rows(p.M, world, rank)
    t = {}
    if p.phi is None:
        from workloads.gpu import gauss_fill
        blk = max(256, ((2 << 30) // (p.N * 4)) // 256 * 256)
        buf = torch.empty((min(blk, rows), p.N), dtype=torch.float32, device=dev)
        cmax = torch.zeros(1, dtype=torch.float32, device=dev)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for r in range(0, rows, blk):
            n = min(blk, rows - r)
            view = buf[:n]
            gauss_fill(view, p.phi_key, p.N, row0 + r, 0, p.phi_sd)
            cmax = torch.maximum(cmax, iht.absmax(view))
        torch.cuda.synchronize()
        t["gen_absmax_ms"] = (time.perf_counter() - t0) * 1e3
    else:
        phi = torch.from_numpy(p.phi[row0:row0 + rows]).to(dev)
        t0 = time.perf_counter()
        cmax = iht.absmax(phi)
        torch.cuda.synchronize()
        t["absmax_ms"] = (time.perf_counter() - t0) * 1e3
    if dist_on:
        import torch.distributed as dist
        dist.all_reduce(cmax, op=dist.ReduceOp.MAX)
    c = float(cmax.item())
    pool = [iht.new_copy(rows, p.N, p.planes, p.b_phi, 0, p.seed, k, c, row_offset=row0, device=dev)
            for k in range(p.K)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    qev = []                       # CUDA event pairs around every quantiser launch (a2)
    if p.phi is None:
        for r in range(0, rows, blk):
            n = min(blk, rows - r)
            view = buf[:n]
            gauss_fill(view, p.phi_key, p.N, row0 + r, 0, p.phi_sd)
            for k0 in range(0, p.K, 8):
                qev.append(_timed(lambda: iht.quantize_rows(view, pool[k0:k0 + 8], r)))
        del buf
    else:
        for k0 in range(0, p.K, 8):
            qev.append(_timed(lambda: iht.quantize_rows(phi, pool[k0:k0 + 8], 0)))
        del phi
    torch.cuda.synchronize()
    t["quantize_wall_ms"] = (time.perf_counter() - t0) * 1e3
    _quantize_stats(t, qev, rows * p.planes * p.N, p.K, p.b_phi)
    torch.cuda.empty_cache()
    return pool, c, t, rows, row0




def _build_pool_cols(p, rank, world, dev, dist_on):
    import torch
    from . import iht
    if p.phi is None:
        raise ValueError("column sharding needs a materialised Phi")
    cols, col0 = shard_cols(p.N, world, rank)
    t = {}
    phi = torch.from_numpy(np.ascontiguousarray(p.phi[:, col0:col0 + cols])).to(dev)   # (M, cols) row-major
    t0 = time.perf_counter()
    cmax = iht.absmax(phi)
    torch.cuda.synchronize()
    t["absmax_ms"] = (time.perf_counter() - t0) * 1e3
    if dist_on:
        import torch.distributed as dist
        dist.all_reduce(cmax, op=dist.ReduceOp.MAX)
    c = float(cmax.item())
    pool = [iht.new_copy(p.M, cols, p.planes, p.b_phi, 0, p.seed, k, c, device=dev, col_offset=col0)
            for k in range(p.K)]
    qev = [_timed(lambda: iht.quantize_rows(phi, pool[k0:k0 + 8], 0)) for k0 in range(0, p.K, 8)]
    _quantize_stats(t, qev, p.M * p.planes * cols, p.K, p.b_phi)
    del phi
    torch.cuda.empty_cache()
    return pool, c, t, p.M, 0


def build_fresh(p, rank, world, dev, dist_on):
    """NEXT-2: this rank's row shard of the fp32 Phi resident on the device (config 4: generated
    block-wise on the device, 64 GiB at one GPU), described for on-the-fly copies.  Returns
    (FreshPhi, c_phi, preprocess timings, rows, row0)."""
    import torch
    from . import iht
    rows, row0 = shard_rows(p.M, world, rank)
    t = {}
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if p.phi is None:
        from workloads.gpu import gauss_fill
        phi = torch.empty((rows, p.N), dtype=torch.float32, device=dev)
        blk = max(256, ((2 << 30) // (p.N * 4)) // 256 * 256)
        for r in range(0, rows, blk):
            n = min(blk, rows - r)
            gauss_fill(phi[r:r + n], p.phi_key, p.N, row0 + r, 0, p.phi_sd)
    else:
        phi = torch.from_numpy(np.ascontiguousarray(p.phi[row0:row0 + rows])).to(dev)
    cmax = iht.absmax(phi)
    if dist_on:
        import torch.distributed as dist
        dist.all_reduce(cmax, op=dist.ReduceOp.MAX)
    c = float(cmax.item())
    torch.cuda.synchronize()
    t["gen_absmax_ms"] = (time.perf_counter() - t0) * 1e3
    return iht.fresh_phi(phi, p.b_phi, 0, p.seed, c, row_offset=row0), c, t, rows, row0
