"""Benchmark: seconds per ALS iteration, Netflix shape (480,189 x 17,770,
99M train ratings, f = 100), on N B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--solver cg16|cg32|exact]
    python bench.py --impl reference ...     # the reference path on the host CPU

A step is one ALS iteration = update-X (CSR, fixed Theta) + update-Theta (CSC,
fixed X) with the ratings and factors resident in HBM; evaluation is excluded
(SURVEY 8(d)).  Default workload = BASELINE configs[2] (approximate batched CG,
fp16 Gram storage); the exact-Cholesky workload (configs[1]) is measured in
the same run on the same data and reported under "exact".  N > 1 runs under
torchrun: users / items are sharded by nnz across ranks and the updated factor
rows are all-gathered over NCCL after each half-update (strong scaling; the
total work is fixed).

Prints ONE JSON line (rank 0).  The reference arm (--impl reference) times the
CPU restatement of the reference path (oracle/, C + OpenMP on every host core)
on a bounded row sample of the same workload and projects it to a full
iteration.
"""

from __future__ import annotations

import argparse
import json
import os
import shutil
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SHAPES = {
    "netflix": (480_189, 17_770, 99_000_000),
    "yahoo": (1_000_990, 624_961, 252_800_000),
    "ml1m": (6_040, 3_706, 1_000_000),
}
SOLVERS = {"cg16": ("cg", "fp16"), "cg32": ("cg", "fp32"), "exact": ("exact", "fp32")}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--shape", default="netflix", choices=list(SHAPES))
    ap.add_argument("--f", type=int, default=100)
    ap.add_argument("--solver", default="cg16", choices=list(SOLVERS))
    ap.add_argument("--gram-kernel", default="auto")
    ap.add_argument("--no-exact", action="store_true", help="skip the configs[1] exact pass")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-ttr", action="store_true", help="skip time-to-RMSE")
    ap.add_argument("--no-next", action="store_true",
                    help="skip the SURVEY 8(f) rows (implicit iteration, eval, build)")
    ap.add_argument("--cpu-sample-nnz", type=int, default=4_000_000)
    return ap.parse_args()


# ----------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index=0):
        self.path = tempfile.mktemp(suffix=".csv")
        self.proc = None
        self.gpu = gpu_index

    def __enter__(self):
        try:
            self.fh = open(self.path, "w")
            # line-buffered so that terminate() loses no samples
            cmd = ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                   "--format=csv,noheader,nounits", "-lms", "20"]
            if shutil.which("stdbuf"):
                cmd = ["stdbuf", "-oL"] + cmd
            self.proc = subprocess.Popen(cmd, stdout=self.fh, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
            return self
        # start the timed region only once sampling is running
        t0 = time.time()
        while time.time() - t0 < 5.0 and self.proc.poll() is None:
            if os.path.getsize(self.path) > 0:
                break
            time.sleep(0.02)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9 and parts[1].isdigit():
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [int(r[1]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        loaded = [s for s in sm if s > 600] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": int(rows[0][2]),
                "samples": len(sm), "power_w_max": max(float(r[3]) for r in rows if r[3] not in ("", "[N/A]")),
                "reasons": reasons}


# ----------------------------------------------------------------- helpers

def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return {"hbm": d["hbm_gbs"], "tensor": d["bf16_tflops"],
                "tensor_sustained": d.get("bf16_tflops_sustained"), "src": "measured",
                "sm_max_mhz": d.get("sm_max_mhz", 1965.0)}
    return {"hbm": 6650.0, "tensor": 1590.0, "tensor_sustained": 1400.0, "src": "fallback",
            "sm_max_mhz": 1965.0}


def traffic_table():
    path = os.path.join(ROOT, "profiles", "traffic.json")
    return json.load(open(path)) if os.path.exists(path) else {}


def workload_label(shape, f, solver, world):
    """Name the BASELINE.json config a run measures (configs[1..4] are the
    Netflix exact / Netflix CG / Yahoo CG / Hugewiki CG workloads)."""
    base = f"{shape}-f{f}-{solver}"
    if shape == "netflix" and f == 100 and solver == "cg16":
        return base + " (BASELINE configs[2])"
    if shape == "netflix" and f == 100 and solver == "exact":
        return base + " (BASELINE configs[1])"
    if shape == "yahoo" and f == 100 and solver == "cg16":
        return base + f" (BASELINE configs[3] shape on {world} GPU{'s' if world > 1 else ''})"
    return base


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def emit(obj, rank):
    if rank == 0:
        print(json.dumps(obj), flush=True)


# ----------------------------------------------------------------- reference arm

def cpu_reference_sample(sr_host, f, method, precision, nnz_budget, nthreads=0):
    """Time the oracle port (C/OpenMP restatement of the reference path) on a
    bounded sample: the first users of the CSR side and the first items of the
    CSC side up to `nnz_budget` ratings each, with the full fixed matrices.
    Returns (projected seconds per full iteration, sample description)."""
    from oracle import oracle as o
    o.lib()
    rng = np.random.default_rng(0)
    out = {}
    total = 0.0
    for side, (ptr, idx, val, nrows, ncols) in (("x", sr_host["csr"]), ("t", sr_host["csc"])):
        k = int(np.searchsorted(ptr, min(nnz_budget, int(ptr[-1])), side="right")) - 1
        k = max(1, min(k, nrows))
        sub_nnz = int(ptr[k])
        fixed = (rng.random((ncols, f), dtype=np.float32) - 0.5) * 0.2
        target = (rng.random((k, f), dtype=np.float32) - 0.5) * 0.2
        view = (ptr[: k + 1], idx[:sub_nnz], val[:sub_nnz], k, ncols)
        o.update_side(view, fixed, target.copy(), 0.05, method, precision, nthreads=nthreads)  # warm
        t0 = time.perf_counter()
        o.update_side(view, fixed, target, 0.05, method, precision, nthreads=nthreads)
        dt = time.perf_counter() - t0
        out[side] = (k, sub_nnz, dt)
        total += dt * (int(ptr[-1]) / sub_nnz)
    desc = (f"oracle port, {o.max_threads()} OpenMP threads: update-X on the first {out['x'][0]} "
            f"users ({out['x'][1]} ratings, {out['x'][2]:.2f}s) + update-Theta on the first "
            f"{out['t'][0]} items ({out['t'][1]} ratings, {out['t'][2]:.2f}s), projected linearly "
            f"in ratings to the full iteration")
    return total, desc, o.max_threads()


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import torch
    m, n, nnz = SHAPES[args.shape]
    method, precision = SOLVERS[args.solver]
    # the same synthetic workload, generated on the host with the reference's
    # own RNG protocol would take minutes at this size; the sample only needs
    # the CSR/CSC structure of the same shape, so draw it directly.
    rng = np.random.default_rng(0)
    per_row = nnz / m
    per_col = nnz / n
    budget = args.cpu_sample_nnz
    ku = max(1, int(budget / per_row))
    kv = max(1, int(budget / per_col))
    deg_u = rng.binomial(n, per_row / n, ku)
    deg_v = rng.binomial(m, per_col / m, kv)
    csr_ptr = np.concatenate([[0], np.cumsum(deg_u)]).astype(np.int64)
    csc_ptr = np.concatenate([[0], np.cumsum(deg_v)]).astype(np.int64)
    csr_idx = np.concatenate([np.sort(rng.choice(n, d, replace=False)) for d in deg_u]).astype(np.int32)
    csc_idx = np.concatenate([np.sort(rng.choice(m, d, replace=False)) for d in deg_v]).astype(np.int32)
    csr_val = rng.standard_normal(csr_ptr[-1]).astype(np.float32)
    csc_val = rng.standard_normal(csc_ptr[-1]).astype(np.float32)
    from oracle import oracle as o
    o.lib()
    f = args.f
    sec = []
    for step in range(args.warmup + args.steps):
        t = 0.0
        for ptr, idx, val, nrows, ncols, full in ((csr_ptr, csr_idx, csr_val, ku, n, m),
                                                   (csc_ptr, csc_idx, csc_val, kv, m, n)):
            fixed = (rng.random((ncols, f), dtype=np.float32) - 0.5) * 0.2
            target = (rng.random((nrows, f), dtype=np.float32) - 0.5) * 0.2
            t0 = time.perf_counter()
            o.update_side((ptr, idx, val, nrows, ncols), fixed, target, 0.05, method, precision)
            t += (time.perf_counter() - t0) * (nnz / int(ptr[-1]))
        if step >= args.warmup:
            sec.append(t)
    v = float(np.median(sec))
    sample = (f"{args.shape} shape f={f} {args.solver}: per step, update-X on {ku} users "
              f"({csr_ptr[-1]} ratings) + update-Theta on {kv} items ({csc_ptr[-1]} ratings) of "
              f"the same degree distribution, projected linearly in ratings to a full iteration")
    cores = o.max_threads()
    print(json.dumps({
        "impl": "reference", "metric": "sec_per_als_iteration", "value": v, "unit": "s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": v * 1e3, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_label(args.shape, f, args.solver, world), "m": m, "n": n, "nnz": nnz,
                   "f": f, "solver": args.solver, "parallelism": "host-cpu"},
        "cpu_baseline": {"value": v, "unit": "s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ----------------------------------------------------------------- our arm

def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    import paper_1808_03843_b200 as cmfb
    from paper_1808_03843_b200 import _native as nat
    from paper_1808_03843_b200 import distributed as cdist

    rank, world, local = dist_env()
    # CMF_DIST_BACKEND=gloo runs the multi-rank flow on a box with fewer GPUs than
    # ranks (ranks share devices; RowGather stages through host memory) -- a
    # functional check only; production runs NCCL, one GPU per rank
    backend = os.environ.get("CMF_DIST_BACKEND", "nccl")
    dev_index = local % torch.cuda.device_count() if backend == "gloo" else local
    torch.cuda.set_device(dev_index)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:
            dist.init_process_group(backend)
    m, n, nnz = SHAPES[args.shape]
    f = args.f
    method, precision = SOLVERS[args.solver]
    solver = cmfb.SolverConfig(method, precision=precision)
    pk = peaks()

    t0 = time.perf_counter()
    train, test = cmfb.gen_synthetic_device(m, n, f, nnz, 0.1, 0.1, seed=0)
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t0
    x0 = torch.from_numpy(cmfb.init_factors(m, f, 0.1, [0, 0])).cuda()
    th0 = torch.from_numpy(cmfb.init_factors(n, f, 0.1, [0, 1])).cuda()

    engine = cdist.ShardedALS(train, f, lam=0.05, solver=solver, gram_kernel=args.gram_kernel,
                              rank=rank, world=world)

    def run_steps(x, th, k, record=None):
        for _ in range(k):
            engine.iteration(x, th, record)

    # ---- warm-up, then the timed region (K iterations, events on the launch stream)
    x, th = x0.clone(), th0.clone()
    exchange = "none (single GPU)" if world == 1 else "NCCL all-gather after each half"
    if world > 1 and os.environ.get("CMF_PEER_STORE", "1") != "0":
        # the fused kernel stores solved rows into every rank's replica (CUDA IPC
        # over NVLink) instead of an all-gather; any setup failure keeps NCCL
        try:
            if engine.attach_replicas(x, th):
                exchange = "peer stores from the fused kernel (CUDA IPC / NVLink), rank barrier per half"
        except Exception as exc:  # noqa: BLE001 - reported in the JSON line
            exchange = f"NCCL all-gather (peer-store setup failed: {exc})"
    run_steps(x, th, args.warmup)
    kern = {}
    nat.LAUNCHES[0] = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev_index) as clk:
        # cudaProfilerStart/Stop bracket the timed region so that
        # `ncu --profile-from-start off` lists exactly the step's launches
        torch.cuda.profiler.start()
        ev0.record()
        run_steps(x, th, args.steps, kern)
        ev1.record()
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    launches = nat.LAUNCHES[0]
    ms_total = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms_total], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms = ms_total / args.steps
    sec = ms / 1e3
    test_rmse = cmfb.rmse(x, th, test)

    # ---- per-kernel device time inside the timed region -> roofline of the dominant kernel
    P = f * (f + 1) // 2
    shard_nnz = engine.local_nnz()
    from paper_1808_03843_b200.als import resolve_events
    per_kernel = {}
    for name, lst in resolve_events(kern).items():
        per_kernel[name] = {"ms_total": sum(lst), "launches": len(lst)}
    gram_ms = sum(v["ms_total"] for k, v in per_kernel.items() if k.startswith("gram"))
    solve_ms = sum(v["ms_total"] for k, v in per_kernel.items() if k.startswith("solve"))
    fused_ms = sum(v["ms_total"] for k, v in per_kernel.items() if k.startswith("fused"))
    gram_flops_step = 2.0 * P * (shard_nnz["x"] + shard_nnz["t"])
    a_bytes = 2 if precision == "fp16" else 4
    nsys = engine.local_rows()
    cg_bytes_step = float((nsys["x"] + nsys["t"]) * (P * a_bytes + 3 * 4 * f))
    gram_tflops = gram_flops_step * args.steps / (gram_ms / 1e3) / 1e12 if gram_ms else 0.0
    solve_gbs = cg_bytes_step * args.steps / (solve_ms / 1e3) / 1e9 if solve_ms else 0.0
    fused_tflops = gram_flops_step * args.steps / (fused_ms / 1e3) / 1e12 if fused_ms else 0.0
    gram_kernel = engine.gram_kernel
    # the committed ncu traffic was captured on the Netflix f=100 CG step
    tt = traffic_table() if (args.shape, f, args.solver) == ("netflix", 100, "cg16") else {}
    dominant = max((fused_ms, "fused"), (gram_ms, "gram"), (solve_ms, "solve"))[1]
    if dominant == "fused":
        roof = {"kernel": "fused_cg_kernel (K1 tcgen05 Gram + K3 CG, A_u never leaves TMEM)",
                "bound": "tensor", "achieved": fused_tflops, "peak": pk["tensor"], "unit": "TFLOP/s",
                "traffic": tt.get("fused_cg_kernel", {}).get("bytes_per_step"),
                "traffic_note": tt.get("fused_cg_kernel", {}).get("note")}
    elif dominant == "gram":
        if gram_kernel.startswith("tc"):
            roof = {"kernel": "gram_tc_kernel (K1)", "bound": "tensor", "achieved": gram_tflops,
                    "peak": pk["tensor"], "unit": "TFLOP/s"}
        else:
            fp32_peak = 148 * 128 * 2 * pk["sm_max_mhz"] * 1e6 / 1e12
            roof = {"kernel": f"gram_simt_{gram_kernel} (K1)", "bound": "fp32-simt",
                    "achieved": gram_tflops, "peak": fp32_peak, "unit": "TFLOP/s",
                    "peak_src": "nominal 148 SM x 128 FP32 lanes x 2 x sm_max_mhz"}
        roof["traffic"] = tt.get("gram")
    else:
        roof = {"kernel": f"{method} solve", "bound": "hbm", "achieved": solve_gbs,
                "peak": pk["hbm"], "unit": "GB/s", "traffic": tt.get("solve")}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["peak_kind"] = pk["src"] + " (burst)"
    roof["units"] = ("K1 algorithmic flops = 2*nnz*f(f+1)/2 per half-update (gram.py:373), "
                     "counted over both halves per step; CG bytes = systems*(P*sizeof(A) + 12f) "
                     "(SURVEY 8(d))")

    result = {
        "metric": "sec_per_als_iteration", "value": sec, "unit": "s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32" + ("/f16-storage" if precision == "fp16" else ""),
        "data": "synthetic (gen_synthetic_device: U[-0.5,0.5) rank-f truth + N(0,0.1) noise, "
                "uniform cells, 10% holdout)",
        "config": {"workload": workload_label(args.shape, f, args.solver, world),
                   "m": m, "n": n, "nnz": train.nnz, "f": f, "lambda": 0.05,
                   "solver": args.solver, "cg_iters": 6, "gram_kernel": gram_kernel,
                   "parallelism": f"rows sharded x{world}" if world > 1 else "single-gpu",
                   "exchange": exchange,
                   "l2": "inputs > L2 (ratings 1.6 GB + Gram workspace)"},
        "gpu_launches": launches,
        "phase_ms_per_step": {"gram": gram_ms / args.steps, "solve": solve_ms / args.steps,
                              "fused_gram_cg": fused_ms / args.steps,
                              "allgather": per_kernel.get("allgather", {}).get("ms_total", 0.0) / args.steps,
                              "peer_barrier": per_kernel.get("peer_barrier", {}).get("ms_total", 0.0)
                              / args.steps},
        "kernels": {"gram_tflops": gram_tflops, "solve_gbs": solve_gbs,
                    "solve_hbm_frac": solve_gbs / pk["hbm"], "fused_tflops": fused_tflops,
                    "per_kernel_ms_per_step": {k: v["ms_total"] / args.steps
                                               for k, v in per_kernel.items()}},
        "roofline": roof,
        "test_rmse_after": test_rmse,
        "gen_seconds": t_gen,
    }

    # ---- clocks seen during the timed region
    result["clocks"] = clk.summary()

    # ---- configs[1]: exact Cholesky on the same data
    if not args.no_exact and method != "exact":
        ex_engine = cdist.ShardedALS(train, f, lam=0.05,
                                     solver=cmfb.SolverConfig("exact"),
                                     gram_kernel="auto", rank=rank, world=world)
        xe, the = x0.clone(), th0.clone()
        for _ in range(2):
            ex_engine.iteration(xe, the)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        kx = {}
        e0.record()
        for _ in range(max(2, args.steps // 2)):
            ex_engine.iteration(xe, the, kx)
        e1.record()
        torch.cuda.synchronize()
        kx = resolve_events(kx)
        ems = e0.elapsed_time(e1) / max(2, args.steps // 2)
        if world > 1:
            te = torch.tensor([ems], dtype=torch.float64, device="cuda")
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
            ems = float(te.item())
        result["exact"] = {"workload": f"{args.shape}-f{f}-exact (BASELINE configs[1])",
                           "sec_per_iteration": ems / 1e3,
                           "gram_ms": sum(sum(v) for k, v in kx.items() if k.startswith("gram")) / max(2, args.steps // 2),
                           "solve_ms": sum(sum(v) for k, v in kx.items() if k.startswith("solve")) / max(2, args.steps // 2),
                           "gram_kernel": ex_engine.gram_kernel,
                           "per_kernel_ms_per_step": {k: sum(v) / max(2, args.steps // 2)
                                                      for k, v in kx.items()}}
        del ex_engine

    # ---- time to RMSE (fresh start; per-epoch eval excluded from the clock)
    # ---- SURVEY 8(f) rows on the same data: implicit ALS iteration (f1, |r| as
    #      the interaction strength, alpha = 40), test RMSE / objective (f2),
    #      CSR + CSC build from device triples (f3); device time, N = 1
    if not args.no_next and world == 1:
        result["next_rows"] = next_rows(cmfb, train, test, x0, th0, m, n)

    if not args.no_ttr and world == 1:
        result["time_to_rmse"] = time_to_rmse(cmfb, engine, train, test, x0, th0, f)

    # ---- e2e through the public API with host buffers (pinned), N = 1
    if not args.no_e2e and world == 1:
        result["e2e"] = e2e(cmfb, train, x0, th0, solver, args)
    else:
        result["e2e"] = None

    # ---- CPU baseline: oracle port on a bounded sample of the same data
    if not args.no_cpu and rank == 0 and world == 1:
        host = {"csr": (train.row_ptr.cpu().numpy(), train.col_idx.cpu().numpy(),
                        train.csr_val.cpu().numpy(), m, n),
                "csc": (train.col_ptr.cpu().numpy(), train.row_idx.cpu().numpy(),
                        train.csc_val.cpu().numpy(), n, m)}
        v, desc, cores = cpu_reference_sample(host, f, method, precision,
                                              args.cpu_sample_nnz)
        result["cpu_baseline"] = {"value": v, "unit": "s", "cores": cores, "kind": "port",
                                  "sample": desc}
    emit(result, rank)
    if world > 1:
        dist.destroy_process_group()


def next_rows(cmfb, train, test, x0, th0, m, n):
    import torch
    from paper_1808_03843_b200.implicit import implicit_update_side, precompute_gram

    def timed(fn, reps):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    out = {}
    users = torch.repeat_interleave(torch.arange(m, device="cuda"), train.row_ptr.diff())
    trip = cmfb.Triples(users, train.col_idx.to(torch.int64), train.csr_val)
    out["build_csr_csc_ms"] = timed(lambda: cmfb.build_device(trip, m, n), 1)
    del users, trip
    x, th = x0.clone(), th0.clone()
    out["test_rmse_ms"] = timed(lambda: cmfb.rmse(x, th, test), 3)
    out["objective_ms"] = timed(lambda: cmfb.objective(x, th, train, 0.05), 3)
    solver = cmfb.SolverConfig("cg")
    csr = cmfb.RowView(train.row_ptr, train.col_idx, train.csr_val.abs(), m, n)
    csc = cmfb.RowView(train.col_ptr, train.row_idx, train.csc_val.abs(), n, m)

    def implicit_iteration():
        implicit_update_side(csr, th, precompute_gram(th), x, 40.0, 0.05, solver, gram_kernel="fma")
        implicit_update_side(csc, x, precompute_gram(x), th, 40.0, 0.05, solver, gram_kernel="fma")

    out["implicit_iteration_ms"] = timed(implicit_iteration, 2)
    out["note"] = ("device time on the bench data; implicit = weighted FMA Gram + CG fp32, "
                   "f_s = 6 (the tensor-core route has no per-rating operand weights yet)")
    return out


def time_to_rmse(cmfb, engine, train, test, x0, th0, f, max_epochs=10):
    import torch
    xe, the = x0.clone(), th0.clone()
    ex_engine = type(engine)(train, f, lam=0.05, solver=cmfb.SolverConfig("exact"),
                             gram_kernel="fma", rank=0, world=1)
    traj_exact = []
    for _ in range(max_epochs):
        ex_engine.iteration(xe, the)
        traj_exact.append(cmfb.rmse(xe, the, test))
    target = traj_exact[-1] + 1e-3
    x, th = x0.clone(), th0.clone()
    cum = 0.0
    traj = []
    reached = None
    for ep in range(max_epochs):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        engine.iteration(x, th)
        e1.record()
        e1.synchronize()
        cum += e0.elapsed_time(e1) / 1e3
        r = cmfb.rmse(x, th, test)
        traj.append(r)
        if reached is None and r <= target:
            reached = (ep + 1, cum)
    return {"target_rmse": target, "target_rule": "exact-path RMSE at epoch 10 + 1e-3",
            "seconds": reached[1] if reached else None, "epochs": reached[0] if reached else None,
            "rmse_trajectory": traj, "exact_trajectory": traj_exact}


def e2e(cmfb, train, x0, th0, solver, args):
    """Same metric through update_side with HOST (pinned) buffers: every step
    copies both views + fixed + target to the device and the target back."""
    import torch
    pin = lambda t: t.cpu().pin_memory()
    csr = cmfb.RowView(pin(train.row_ptr), pin(train.col_idx), pin(train.csr_val), train.m, train.n)
    csc = cmfb.RowView(pin(train.col_ptr), pin(train.row_idx), pin(train.csc_val), train.n, train.m)
    x, th = pin(x0), pin(th0)
    h2d = sum(t.numel() * t.element_size() for t in (*csr[:3], *csc[:3])) + 2 * (
        x.numel() + th.numel()) * 4
    d2h = (x.numel() + th.numel()) * 4
    steps = max(2, args.steps // 2)
    for _ in range(1):
        cmfb.update_side(csr, th, x, 0.05, solver, gram_kernel=args.gram_kernel)
        cmfb.update_side(csc, x, th, 0.05, solver, gram_kernel=args.gram_kernel)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        cmfb.update_side(csr, th, x, 0.05, solver, gram_kernel=args.gram_kernel)
        cmfb.update_side(csc, x, th, 0.05, solver, gram_kernel=args.gram_kernel)
    torch.cuda.synchronize()
    v = (time.perf_counter() - t0) / steps
    return {"value": v, "unit": "s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "pcie_gbs": (h2d + d2h) / v / 1e9,
            "api": "paper_1808_03843_b200.update_side x2 (C ABI via ctypes), pinned host buffers; "
                   "copies of chunk k+1 / k-1 overlap the fused kernel on chunk k"}


if __name__ == "__main__":
    main()
