#!/usr/bin/env python
"""bench.py -- low-precision IHT (arXiv 1802.04907) hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Metric (BASELINE.json): IHT iter/s and Phi-stream HBM GB/s (% of peak).
A "step" is one complete QNIHT solve of one observation y: quantise y (a3), then
n* iterations of forward (a4) -> adjoint (a5) -> [NCCL all-reduce of g] ->
update + H_s (a6), over a pool of K pre-quantised copies of Phi.  Phi's scale
and quantisation (a1, a2) are one-time per-operator preprocessing (the paper
quantises to cut transmission from storage) and are reported under
"preprocess".  value = steps * n* / (max over ranks of the device time).

Default workload: BASELINE config 4 (real Gaussian 65536 x 262144, 4-bit Phi,
8-bit y, s = 1024, n* = 100, K = 2 copies = 16 GiB of codes per GPU at N = 1,
row-sharded at N > 1).  The pool exceeds the 126 MB L2, so every iteration
streams its adjoint copy from HBM (no L2 flush needed); a pool that fits L2 (config 1)
is timed step by step with an L2 flush before each step, outside the timed events.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PAPER_CONTEXT = "paper: CPU 4-bit 4.19x / 8-bit 2.84x vs 32-bit (Haswell E3-1285L v3, P:587); " \
                "FPGA 2&8-bit 9.19x to 90% support (P:578) -- context only, other hardware"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--bits", type=int, default=None, help="override b_Phi (2/4/8 sweep)")
    ap.add_argument("--K", type=int, default=None, help="pool of quantised copies")
    ap.add_argument("--variant", type=int, default=0, help="adjoint: 0 int8 MMA, 1 FFMA")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--adaptive", action="store_true", help="Algorithm 1's adaptive step (NEXT-1)")
    ap.add_argument("--fresh", action="store_true",
                    help="NEXT-2: fresh copies drawn on the fly from the resident fp32 Phi (K = 2 n*, no codes)")
    return ap.parse_args()


def measured_tensor_peak_int8():
    """Dense int8 tensor peak (TOP/s): the measured bf16 peak x the nominal int8/bf16 ratio
    (4.5 / 2.25 = 2, B200_PROFILING.md).  Burst figure: the kernel is timed per launch."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return 2.0 * float(d["bf16_tflops"]), "measured bf16 x 2 (nominal int8/bf16 ratio)"
    except Exception:
        return 4500.0, "nominal"


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id):
        self.gpu_id = gpu_id
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu_id}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100", "-f", self.path],
                                         stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.25)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        self.proc.wait()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 8:
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[4:8]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------------------------- problem setup
L2_FLUSH_BYTES = 256 << 20      # > the 126 MB L2 of a B200


def make_problem(args):
    from workloads import gen as G
    p = G.config_problem(args.config, K=args.K, b_phi=args.bits)
    if args.config == 4 and args.K is None:
        p.K = 2
    return p


# ----------------------------------------------------------------------------- CPU oracle
def oracle_sample(p, steps=None):
    """Time the float64 oracle (as it stands) on bounded samples of the workload: the
    first R0 and 2*R0 measurement rows (all N columns), K = 1 copy (the same
    forward/adjoint work per iteration as K = 2, half the one-time quantisation),
    n iterations each, with the copies pre-quantised (one-time preprocess, excluded
    as on the GPU).  Per-iteration time is fitted as t(rows) = a + b rows and
    extrapolated to the full M rows."""
    import numpy as np
    from oracle import iht as OI
    from oracle import quantize as OQ
    try:
        from threadpoolctl import threadpool_info
        threads = max([d.get("num_threads", 1) for d in threadpool_info()] or [1])
    except Exception:
        threads = os.cpu_count()
    r0 = max(1, min(p.M // 2, (1 << 23) // (p.N * p.planes)))
    r0 = 1 << int(np.floor(np.log2(r0)))
    n_it = 3 if steps is None else max(1, steps)
    B = p.meta.get("batch_y").shape[1] if "batch_y" in p.meta else 1
    times = []
    for rows in (r0, 2 * r0):
        phi = p.phi_rows(0, rows)
        y = p.meta["batch_y"][:rows, 0] if B > 1 else p.y[:rows]
        pool = OI.CopyPool(phi, p.b_phi, 0, p.seed, OQ.scale_c(phi), cache=2)
        pool.dequantized(0)                                   # one-time preprocess
        t0 = time.perf_counter()
        OI.qniht(phi, y, p.s, n_it, p.mu, p.b_phi, p.b_y, p.seed, 1, record=False, pool=pool)
        times.append((time.perf_counter() - t0) / n_it)
    b = max((times[1] - times[0]) / r0, 0.0)
    a = max(times[0] - b * r0, 0.0)
    per_iter = (a + b * p.M) * B
    return {"value": 1.0 / per_iter, "unit": "iter/s", "cores": threads, "kind": "oracle",
            "sample": f"rows 0..{r0 - 1} and 0..{2 * r0 - 1} of {p.M}, all {p.N} columns, K=1 copy, "
                      f"{n_it} float64 iterations each (copy quantisation excluded); per-iteration time "
                      f"fitted a + b*rows ({times[0] * 1e3:.1f} / {times[1] * 1e3:.1f} ms) and extrapolated "
                      f"to {p.M} rows" + (f", one snapshot timed and multiplied by the batch B={B} "
                                          f"(the oracle runs snapshots independently)" if B > 1 else ""),
            "host_cores": os.cpu_count()}


# ----------------------------------------------------------------------------- main
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world == 1 and args.gpus > 1:
        print(json.dumps({"error": "--gpus N>1 must be launched with torchrun"}))
        return 2

    if args.impl == "reference":
        if rank != 0:
            return 0
        p = make_problem(args)
        for _ in range(max(0, args.warmup)):
            pass
        cb = oracle_sample(p, steps=max(1, args.steps))
        line = {"impl": "reference", "metric": "IHT iter/s", "value": cb["value"], "unit": "iter/s",
                "n_gpus": 0, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": p.name, "M": p.M, "N": p.N, "b_phi": p.b_phi, "s": p.s,
                           "n_iter": p.n_iter},
                "cpu_baseline": cb,
                "e2e": {"value": cb["value"], "unit": "iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return 0

    import torch
    from paper_1802_04907_b200 import iht

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist_on = world > 1
    comm = None
    if dist_on:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        comm = iht.Comm(rank, world, local)

    def barrier():
        if dist_on:
            torch.distributed.barrier(device_ids=[local])

    def max_over_ranks(v):
        if not dist_on:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    t_setup = time.perf_counter()
    p = make_problem(args)
    B = p.meta["batch_y"].shape[1] if "batch_y" in p.meta else 1
    from paper_1802_04907_b200.problem import build_fresh, build_pool
    if args.fresh:
        if B > 1:
            raise SystemExit("--fresh is the single-observation path")
        pool, c_phi, prep, rows, row0 = build_fresh(p, rank, world, dev, dist_on)
    else:
        pool, c_phi, prep, rows, row0 = build_pool(p, rank, world, dev, dist_on, shard="cols" if B > 1 else "rows")
    if B > 1:        # (B, M) observations, replicated on every column shard
        y_shard = np.ascontiguousarray(p.meta["batch_y"].T)
    else:
        y_shard = p.y[row0:row0 + rows]
    y_dev = torch.from_numpy(y_shard).to(dev)
    # the timed solver has no profiling events in its graph (they would separate the kernels
    # and defeat programmatic dependent launch); a second, profiled solver over the same
    # pool times the adjoint launches for the roofline after the timed region
    sol = iht.Solver(pool, p.s, p.n_iter, p.mu, p.b_y, p.seed, adjoint_variant=args.variant, comm=comm,
                     profile=False, nrhs=B, adaptive=args.adaptive)
    setup_s = time.perf_counter() - t_setup

    # ---- device-resident timed region -----------------------------------------------
    _ncols = pool.desc.cols if args.fresh else pool[0].cols
    copy_bytes_est = (4 * rows * _ncols * p.planes if args.fresh
                      else iht._lib.load().iht_qmat_bytes(rows, _ncols, p.planes, p.b_phi))
    for _ in range(max(3, args.warmup)):
        sol.run(y_dev)
    torch.cuda.synchronize()
    barrier()
    props = torch.cuda.get_device_properties(local)
    gpu_id = getattr(props, "uuid", None)
    gpu_id = f"GPU-{gpu_id}" if gpu_id is not None and not str(gpu_id).startswith("GPU-") else (gpu_id or local)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    resident = (copy_bytes_est if args.fresh else p.K * copy_bytes_est) <= L2_FLUSH_BYTES

    def timed_region():
        clk = ClockSampler(gpu_id if gpu_id else local)
        clk.start()
        torch.cuda.synchronize()
        barrier()
        if not resident:
            # the pool exceeds L2: every iteration streams its copies from HBM
            e0.record()
            for _ in range(args.steps):
                sol.run(y_dev)
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1)
        else:
            # the pool would stay in L2 across steps: flush L2 (write a buffer larger than
            # it) before every step, outside the timed events, and sum the per-step times
            flush = torch.empty(L2_FLUSH_BYTES // 4 * 2, dtype=torch.float32, device=dev)
            t = 0.0
            for _ in range(args.steps):
                flush.fill_(1.0)
                e0.record()
                sol.run(y_dev)
                e1.record()
                torch.cuda.synchronize()
                t += e0.elapsed_time(e1)
            del flush
        barrier()
        return t, clk.stop()

    ms_dev, clocks = timed_region()
    # a hardware / thermal slowdown during the timed region invalidates it: measure once more
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    if max_over_ranks(1.0 if bad & set(clocks.get("reasons") or []) else 0.0) > 0.0:   # all ranks agree
        first = clocks
        ms_dev, clocks = timed_region()
        clocks = dict(clocks, remeasured_after=sorted(bad & set(first.get("reasons") or [])) or ["another rank"])
    ms = max_over_ranks(ms_dev)
    sol_prof = iht.Solver(pool, p.s, p.n_iter, p.mu, p.b_y, p.seed, adjoint_variant=args.variant, comm=comm,
                          profile=True, nrhs=B, adaptive=args.adaptive)
    for _ in range(2):
        sol_prof.run(y_dev)
    torch.cuda.synchronize()
    adj_ms = sol_prof.adjoint_times_ms()
    sol_prof.close()
    out_idx, out_val, out_nnz = sol.out_idx, sol.out_val, sol.out_nnz
    nnz = [int(v) for v in out_nnz.cpu()]
    if min(nnz) < 0:   # a poisoned (non-finite) iterate lets kernels exit early: not a valid run
        raise SystemExit(f"bench: the iteration diverged (support size {min(nnz)}): step mu = {p.mu} "
                         "is unstable for this workload (reading c9)")
    launches_per_run = sol.launches_per_run()

    # ---- end-to-end through the public API with host buffers --------------------------
    e2e = None
    if not args.no_e2e:
        y_pin = torch.from_numpy(y_shard.copy()).pin_memory()
        oshape = (B, p.s) if B > 1 else (p.s,)
        oi = torch.empty(oshape, dtype=torch.int32).pin_memory()
        ov = torch.empty(oshape, dtype=torch.float32).pin_memory()
        on = torch.empty(B, dtype=torch.int32).pin_memory()
        sol.run_host(y_pin, oi, ov, on)
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            sol.run_host(y_pin, oi, ov, on)
        e2e_s = max_over_ranks(time.perf_counter() - t0)
        yb = y_pin.numel() * y_pin.element_size() * (2 if y_pin.is_complex() else 1)
        e2e = {"value": args.steps * p.n_iter / e2e_s, "unit": "iter/s",
               "h2d_bytes_per_step": int(yb), "d2h_bytes_per_step": int(B * (p.s * 8 + 4)),
               "path": "iht_solver_run(IHT_HOST_IO): pinned y -> device, solve, x -> pinned host, sync"}

    # ---- bookkeeping --------------------------------------------------------------------
    peak, peak_kind = measured_peaks()
    ncols = pool.desc.cols if args.fresh else pool[0].cols     # this rank's columns
    strip = iht.strip_bytes(rows, p.planes, p.b_phi)
    copy_bytes = iht._lib.load().iht_qmat_bytes(rows, ncols, p.planes, p.b_phi)
    if args.fresh:          # the adjoint streams the fp32 Phi (4 bytes per component), the forward s columns
        copy_bytes = 4 * rows * ncols * p.planes
        strip = 4 * rows * p.planes
    R = iht.vec_len(rows, p.planes)
    adj_bytes = copy_bytes + B * (4 * R + 4 * ncols)          # codes + r read + g write
    fwd_bytes = B * (p.s * strip + 4 * R + 4 * R)              # support strips + yhat + r
    thr_bytes = B * (4 * ncols * 2 + 8 * p.s)                  # g read + a write (+ x)
    iter_bytes = adj_bytes + fwd_bytes + thr_bytes
    iters = args.steps * p.n_iter
    value = iters / (ms / 1e3)
    adj_avg = statistics.mean(adj_ms)
    adj_gbs = adj_bytes / (adj_avg / 1e3) / 1e9
    stream_gbs = iter_bytes * iters / (ms / 1e3) / 1e9     # per GPU
    traffic = None
    tp = os.path.join(ROOT, "profiles", "adjoint_traffic.json")
    if os.path.exists(tp):
        try:
            d = json.load(open(tp))
            key = f"{p.name}:b{p.b_phi}:gpus{world}:v{args.variant}"
            traffic = d.get(key)
        except Exception:
            traffic = None
    if B > 1:   # (a7) tensor-core bound: algorithmic int8 ops 2 R N B (one multiply-add per code per snapshot)
        tpeak, tpeak_kind = measured_tensor_peak_int8()
        adj_ops = 2.0 * R * ncols * B
        roof = {"bound": "tensor", "kernel": "adjoint_batched_kernel (+ batched_limbs_kernel)",
                "achieved": adj_ops / (adj_avg / 1e3) / 1e12, "peak": tpeak, "unit": "TOP/s",
                "frac": adj_ops / (adj_avg / 1e3) / 1e12 / tpeak, "peak_kind": tpeak_kind,
                "traffic": traffic, "traffic_unit": "DRAM bytes per launch (ncu --set full)",
                "algorithmic_ops_per_launch": adj_ops,
                "executed_int8_ops_per_launch": 2 * adj_ops, "avg_launch_ms": adj_avg,
                "launches_timed": len(adj_ms), "code_bytes_per_launch": copy_bytes,
                "how": "CUDA event pair around every batched adjoint (limb prep + tcgen05 GEMM) inside a "
                       "profiled copy of the solver graph (run after the timed region); ops = 2 R N B useful (x2 executed: two int8 limbs of r)"}

    if rank != 0:
        return 0
    cb = None
    if not args.no_cpu_baseline and world == 1:
        cb = oracle_sample(p)
    line = {
        "metric": "IHT iter/s (Phi-stream HBM GB/s, % of peak)",
        "value": value,
        "unit": "iter/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": max(3, args.warmup),
        "ms_per_step": ms / args.steps,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": ("u8 x s8 -> s32 tcgen05 (kind::i8) batched adjoint" if B > 1 else
                  "s8/s32 int8-MMA adjoint") + ", f32 forward/update",
        "data": "synthetic",
        "config": {
            "workload": f"{p.name}: {'complex radio' if p.complex else 'real Gaussian'} {p.M}x{p.N}, "
                        f"{p.b_phi}-bit Phi, {p.b_y}-bit y, s={p.s}, n*={p.n_iter}, mu={p.mu:g}, K={p.K} copies"
                        + (f", B={B} snapshots per iteration (one iter = all B)" if B > 1 else ""),
            "M": p.M, "N": p.N, "b_phi": p.b_phi, "b_y": p.b_y, "s": p.s, "n_iter": p.n_iter, "K": p.K,
            "batch": B,
            "parallelism": (f"column-sharded x{world}" + (", NCCL all-reduce of r + all-gather of top-s candidates"
                                                          if world > 1 else "") if B > 1 else
                            f"row-sharded x{world}" + (", NCCL all-reduce of g per iteration" if world > 1 else "")),
            "l2": (lambda res: f"inputs > L2: {res / 2**30:.2f} GiB per GPU streamed from HBM" if not resident
                   else f"pool {res / 2**20:.1f} MiB fits L2: L2 flushed (256 MiB write) before every timed step, "
                        "per-step event times summed")(copy_bytes if args.fresh else p.K * copy_bytes),
            "adjoint_variant": args.variant,
            "step": "adaptive mu-hat with accept/shrink loop (Algorithm 1, P:350-363)" if args.adaptive
                    else f"fixed mu = {p.mu:g}",
            "copies": "fresh: drawn on the fly from the resident fp32 Phi, K = 2 n* (NEXT-2)" if args.fresh
                      else f"pool of K = {p.K} stored quantised copies",
        },
        "hbm": {"phi_stream_GBps_per_gpu": stream_gbs, "frac_of_measured": stream_gbs / peak,
                "frac_of_8TBps": stream_gbs / 8000.0, "bytes_per_iter_per_gpu": iter_bytes},
        "roofline": roof if B > 1 else
                    {"bound": "hbm", "kernel": "adjoint_fresh_kernel (fp32 Phi + Philox, NEXT-2)" if args.fresh else
                               "adjoint_mma_kernel" if args.variant == 0 else "adjoint_ffma_kernel",
                     "achieved": adj_gbs, "peak": peak, "unit": "GB/s", "frac": adj_gbs / peak,
                     "peak_kind": peak_kind, "traffic": traffic,
                     "algorithmic_bytes_per_launch": adj_bytes, "avg_launch_ms": adj_avg,
                     "launches_timed": len(adj_ms),
                     "how": "CUDA event pair around every adjoint inside a profiled copy of the solver graph, run after the timed region"},
        "cpu_baseline": cb,
        "e2e": e2e,
        "gpu_launches": int(launches_per_run * args.steps),
        "clocks": clocks,
        "preprocess": {**prep, "c_phi": c_phi, "setup_s": setup_s},
        "result": {"support_size": nnz if B > 1 else nnz[0]},
        "snapshot_iter_per_s": value * B,
        "context": PAPER_CONTEXT,
    }
    print(json.dumps(line))
    sys.stdout.flush()
    if comm is not None:
        comm.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
