#!/usr/bin/env python
"""Benchmark of the randomized-LUPP skeleton-selection hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--k 512] [--impl ours|reference]

Workload (BASELINE.json configs[1], "C2"): A = U diag(10^(-i/50)) V^T, 4096 x 4096 FP64,
Haar U, V (seed 1002); Gaussian Omega, k = 512, l = k + 10 = 522 (seed 2002 + k).
One step = the whole hot path of SURVEY.md section 8(a) for C2:
    S0+S1 sketch X = Omega A  ->  S2 select_cols (LUPP)  ->  S2' select_cols_cpqr (comparison)
    ->  S5 id_coeffs  ->  S6 residual ||A - CC^+A||_F (gather S3 + LUPP-basis S4 inside).
The other configs follow their SURVEY 8(d) path: C3 / C4 add S3 gather + S4 select_rows as
stages and take the CUR (C3) / column- and row-ID (C4) residuals; S2' runs on C2 only.
value = the BASELINE.json metric "skeleton-selection time (sketch+LUPP)" = S1 + S2 device time
per step (ms, lower is better), max over ranks.  ms_per_step = the whole step.
L2 policy: a 512 MiB buffer is overwritten between timed steps (untimed), so every step
starts cold; per-step CUDA events on the library's stream.

--impl reference times the plain CPU oracle (oracle/) on the same config on the host cores
(the reference arm for this paper-only build).
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAK_TFLOPS = 37.13   # measured DMMA issue ceiling on this pool's B200 (profiles/round1/fp64_peaks.txt)
L2_FLUSH_BYTES = 512 << 20


def hbm_peak_gbs():
    """(GB/s, source): MEASURED_PEAKS.json's copy bandwidth, else the profiling guide's fallback."""
    try:
        v = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
        return v, "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--k", type=int, default=None, help="default: C1 20, C2 512, C3 500, C4 200, C5 1000")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--piter", type=int, default=0, help="plain power iterations (Rand-LUPP-qpiter, P:527)")
    ap.add_argument("--dist-exchange", default="replicate", choices=["replicate", "step", "p2p"],
                    help="N > 1: column-LUPP exchange -- one k x n all-gather then replicated LUPP, one "
                         "all-gather of P records per pivot step (CUDA graph), or the records stored into "
                         "the peers' mailboxes by the step kernel itself (NVLink peer memory, CUDA graph)")
    return ap.parse_args()


def workload(args):
    from inputs import CONFIGS
    cfg = CONFIGS[args.config]
    if args.k is None:
        args.k = {"C1": 20, "C2": 512, "C3": 500, "C4": 200, "C5": 1000}[args.config]
        if getattr(args, "piter", 0) and args.config == "C2":
            # X = Omega (A^T A)^q squares the C2 spectrum (10^(-i/25)): beyond k ~ 390 the sketch is
            # rank deficient at LUPP's 1e-14 threshold (both the oracle and the GPU stop there)
            args.k = 256
    k = args.k
    l = cfg["l"](k)
    seed = cfg["sk_seed"] + (k if args.config in ("C2", "C4") else 0)
    desc = {
        "C2": f"C2: A 4096x4096 FP64 = U diag(10^(-i/50)) V^T (Haar), Gaussian Omega, k={k}, l={l}",
        "C5": f"C5: A 131072x65536 FP64 (68.7 GB) = U diag(i^-1.5) V^T, U,V products of 64 Householder "
              f"reflectors, built on the device; Gaussian Omega, k={k}, l={l}",
    }.get(args.config, f"{args.config} k={k} l={l}")
    if getattr(args, "piter", 0):
        desc += f", {args.piter} plain power iteration(s) X = Omega (A^T A)^q (Rand-LUPP-{args.piter}piter)"
    return cfg, k, l, seed, desc


def make_input(args, cfg):
    from inputs import make_config
    A, sigma = make_config(args.config, seed=cfg["seed"])
    return A, sigma


def cpu_info():
    cores = len(os.sched_getaffinity(0))
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return cores, model


def oracle_selection(A, k, l, seed, emb="gaussian", piter=0):
    """The oracle's sketch (with q = piter plain power iterations) + LUPP (test infrastructure;
    timed as the CPU baseline)."""
    from oracle import lupp as o_lupp
    from oracle import sketch as o_sketch
    X = o_sketch.sketch(A, l, emb, seed) if piter == 0 else o_sketch.sketch_power(A, l, emb, seed, piter)
    piv, _, _, _ = o_lupp.select_cols(X, k)
    return piv


class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.QUERY}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.rows = []
        if self.proc is None:
            return
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=5)
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def summary(self):
        if not getattr(self, "rows", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[5 + i].lower() == "active"})
        busy = [s for s in sm if s > 500] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def run_reference(args):
    """--impl reference: the oracle on the host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg, k, l, seed, desc = workload(args)
    if args.config == "C5":   # 68.7 GB: the host oracle cannot hold it (the GPU path builds it on device)
        print(json.dumps({"impl": "reference", "unavailable": "C5 (131072 x 65536 FP64, 68.7 GB) exceeds the "
                          "host oracle's memory; the reference arm runs C1-C4"}), flush=True)
        return 0
    A, _ = make_input(args, cfg)
    cores, model = cpu_info()
    steps = max(1, min(args.steps, 3))
    warm = min(args.warmup, 1)
    for _ in range(warm):
        oracle_selection(A, k, l, seed, cfg["emb"], args.piter)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        oracle_selection(A, k, l, seed, cfg["emb"], args.piter)
        times.append((time.perf_counter() - t0) * 1e3)
    v = statistics.mean(times)
    line = {
        "impl": "reference", "metric": "skeleton-selection time (sketch+LUPP)", "value": v, "unit": "ms",
        "n_gpus": args.gpus, "steps": steps, "warmup": warm, "ms_per_step": v, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": desc, "m": int(A.shape[0]), "n": int(A.shape[1]), "k": k, "l": l},
        "cpu_baseline": {"value": v, "unit": "ms", "cores": cores, "kind": "oracle",
                         "sample": f"full {args.config} selection (oracle sketch{' with %d power iteration(s)' % args.piter if args.piter else ''} + LUPP) on {model}"},
        "e2e": {"value": v, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main_dist(args, world, rank, local):
    """N > 1 GPUs (torchrun): the column-sharded path of SURVEY 8(e), weak scaling.

    Rank r holds a 4096 x 4096 C2-type block (own Haar factors, seed 1002 + r), so the global A is
    4096 x 4096N.  One step = sketch of the local block (Omega regenerated from the seed, no
    communication) -> all-gather of the k LUPP-visible sketch rows -> column LUPP on the full panel
    (replicated, identical J_s on every rank) -> C = A(:, J_s) by a sum all-reduce -> column-ID
    residual (local squared sums + all-reduce).  value = sketch + selection time, max over ranks."""
    import torch
    import torch.distributed as dist

    import paper_2104_05877_b200 as sk
    from inputs import make_c2
    from paper_2104_05877_b200.dist import _all_gather_cols

    dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(dev)
    k = args.k if args.k is not None else 512              # C2's bench k
    l = k + 10
    seed = 2002 + k
    A_np, _ = make_c2(seed=1002 + rank)
    m, nloc = A_np.shape
    n_global = nloc * world
    col0 = rank * nloc
    with torch.cuda.stream(stream):
        A = sk.fortran(torch.from_numpy(np.ascontiguousarray(A_np)).to(dev))
        flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
        Xbuf = torch.empty((l, nloc), dtype=torch.float64, device=dev)
    torch.cuda.synchronize(dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    cap = []

    def step(record):
        e = [ev() for _ in range(5)]
        e[0].record(stream)
        X = sk.sketch(A, l, "gaussian", seed, out=Xbuf)
        e[1].record(stream)
        if args.dist_exchange == "step":
            if not cap:
                from paper_2104_05877_b200.dist import CapturedStepwise
                cap.append(CapturedStepwise(Xbuf, n_global, k))
            Js, _, _ = cap[0].run()
        elif args.dist_exchange == "p2p":
            if not cap:                      # mailboxes + one captured graph of begin + k steps
                from paper_2104_05877_b200.dist import P2PStepwise
                p2p = P2PStepwise(n_global, k, None, local)
                p2p.run(Xbuf)
                torch.cuda.synchronize(dev)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    p2p.sel.begin(Xbuf)
                    for t in range(1, k + 1):
                        p2p.sel.step(t)
                cap.append((p2p, g))
            cap[0][1].replay()
            Js = cap[0][0].sel.Js
        else:
            Xk = _all_gather_cols(X[:k], n_global, None, world)
            Js, _, _, _ = sk.select_cols(Xk, k, check=False)
        e[2].record(stream)
        C = sk.gather_cols_shard(A, Js, col0)
        Ct = C.t().contiguous()
        dist.all_reduce(Ct)
        e[3].record(stream)
        r2, a2 = sk.residual_cols(A, Ct.t())
        sums = torch.tensor([r2, a2], dtype=torch.float64, device=dev)
        dist.all_reduce(sums)
        e[4].record(stream)
        record(e)
        return Js, sums

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step(lambda e: None)
        torch.cuda.synchronize(dev)
        dist.barrier()
        recs = []
        launches0 = sk.launch_count(local)
        with ClockSampler(local) as clk:
            torch.cuda.synchronize(dev)
            for _ in range(args.steps):
                flush.fill_(1)
                out = step(recs.append)
            torch.cuda.synchronize(dev)
        launches = sk.launch_count(local) - launches0
        dist.barrier()
    sk_ms = statistics.mean(e[0].elapsed_time(e[1]) for e in recs)
    sel_ms = statistics.mean(e[0].elapsed_time(e[2]) for e in recs)
    step_ms = statistics.mean(e[0].elapsed_time(e[4]) for e in recs)
    t = torch.tensor([sel_ms, step_ms, sk_ms], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    sel_ms, step_ms, sk_ms_max = float(t[0]), float(t[1]), float(t[2])
    Js, sums = out
    achieved = 2.0 * l * m * nloc / (sk_ms * 1e-3) / 1e12
    # end to end: pinned host block -> device (inside the timed region) -> sketch -> selection -> J_s on host
    e2e = None
    if not args.no_e2e:
        A_host = torch.from_numpy(np.ascontiguousarray(A_np.T)).pin_memory()      # rows = columns of A
        A_dev = torch.empty_like(A_host, device=dev)
        times = []
        with torch.cuda.stream(stream):
            for it in range(2 + max(3, min(args.steps, 10))):
                e0, e1 = ev(), ev()
                e0.record(stream)
                A_dev.copy_(A_host, non_blocking=True)
                Ad = A_dev.t()
                X = sk.sketch(Ad, l, "gaussian", seed)
                Xk = _all_gather_cols(X[:k], n_global, None, world)
                Js_d, _, _, _ = sk.select_cols(Xk, k, check=False)
                Js_h = Js_d.cpu()
                e1.record(stream)
                e1.synchronize()
                if it >= 2:
                    times.append(e0.elapsed_time(e1))
        t = torch.tensor([statistics.mean(times)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e = {"value": float(t[0]), "unit": "ms", "h2d_bytes_per_step": int(m * nloc * 8),
               "d2h_bytes_per_step": int(k * 8), "api": "dist path (torch.distributed + libskel.so), host A block per rank"}
    if rank == 0:
        line = {
            "metric": "skeleton-selection time (sketch+LUPP)", "value": sel_ms, "unit": "ms",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"C2-type blocks: A 4096 x {n_global} FP64 column-sharded, 4096 x 4096 "
                                   f"U diag(10^(-i/50)) V^T per rank, Gaussian Omega, k={k}, l={l}",
                       "m": m, "n": n_global, "k": k, "l": l, "parallelism": f"column-sharded x{world}", "lupp_exchange": args.dist_exchange,
                       "l2": "flushed: 512 MiB overwrite between timed steps (untimed)"},
            "residual": {"col_id_fro": math.sqrt(max(float(sums[0]), 0.0)), "normA_fro": math.sqrt(float(sums[1]))},
            "roofline": {"kernel": "sk_sketch Gaussian = k_omega_image + k_sketch_pre (+ split-K reduce)", "bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS,
                         "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS, "traffic": None},
            "cpu_baseline": None, "e2e": e2e, "gpu_launches": int(launches), "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1 or os.environ.get("SKEL_BENCH_DIST") == "1":
        return main_dist(args, int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
                         int(os.environ.get("LOCAL_RANK", "0")))

    import torch
    import torch.distributed as dist

    import paper_2104_05877_b200 as sk

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(dev)

    cfg, k, l, seed, desc = workload(args)
    emb = cfg["emb"]
    with torch.cuda.stream(stream):
        if args.config == "C5":          # 68.7 GB: built on the device (inputs/c5.py), no host copy
            from inputs.c5 import build_on_device
            A, sigma = build_on_device(dev)
            A_np = None
            m, n = A.shape
        else:
            A_np, sigma = make_input(args, cfg)
            m, n = A_np.shape
            A = sk.fortran(torch.from_numpy(np.ascontiguousarray(A_np)).to(dev))
        flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    torch.cuda.synchronize(dev)

    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    # the step follows each configuration's path in SURVEY 8(d): S2' (CPQR) on C2, S3 + S4 (gather,
    # row LUPP) on C3 / C4, the residual kinds per config (CUR on C3, column and row ID on C4)
    do_cpqr = args.config == "C2"
    do_rows = args.config in ("C3", "C4")
    res_kinds = {"C3": ["cur"], "C4": ["col_id", "row_id"]}.get(args.config, ["col_id"])
    stage_names = (["sketch", "select_cols_lupp"] + (["select_cols_cpqr"] if do_cpqr else [])
                   + (["gather_cols", "select_rows_lupp"] if do_rows else []) + ["id_coeffs", "residual"])

    def step(record):
        """One pass of the hot path; record(events), one event per stage boundary."""
        e = [ev() for _ in range(len(stage_names) + 1)]
        nxt = iter(e[1:])
        e[0].record(stream)
        X = (sk.sketch(A, l, emb, seed, cfg.get("zeta", 8)) if args.piter == 0
             else sk.sketch_power(A, l, emb, seed, args.piter, cfg.get("zeta", 8)))
        next(nxt).record(stream)
        Js, Lf, _, _ = sk.select_cols(X, k, check=False)
        next(nxt).record(stream)
        Jc = Is = None
        if do_cpqr:
            Jc, _ = sk.select_cols_cpqr(X, k, check=False)
            next(nxt).record(stream)
        if do_rows:
            C = sk.gather_cols(A, Js)
            next(nxt).record(stream)
            Is, _, _, _ = sk.select_rows(C, k, want_factors=False, check=False)
            next(nxt).record(stream)
        Z, _ = sk.id_coeffs(Lf, Js)
        next(nxt).record(stream)
        res = {kind: sk.residual(A, Js, Is, kind) for kind in res_kinds}
        next(nxt).record(stream)
        record(e)
        return Js, Jc, res

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step(lambda e: None)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        recs = []
        launches0 = sk.launch_count(local)
        with ClockSampler(local) as clk:
            torch.cuda.synchronize(dev)
            for _ in range(args.steps):
                flush.fill_(1)                     # untimed L2 flush between steps
                out = step(recs.append)
            torch.cuda.synchronize(dev)
        launches = sk.launch_count(local) - launches0
        if world > 1:
            dist.barrier()
    stage_ms = {nm: [] for nm in stage_names}
    step_ms = []
    for e in recs:
        for i, nm in enumerate(stage_names):
            stage_ms[nm].append(e[i].elapsed_time(e[i + 1]))
        step_ms.append(e[0].elapsed_time(e[-1]))
    sel = [a + b for a, b in zip(stage_ms["sketch"], stage_ms["select_cols_lupp"])]
    value = statistics.mean(sel)
    ms_step = statistics.mean(step_ms)
    if world > 1:
        t = torch.tensor([value, ms_step], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        value, ms_step = float(t[0]), float(t[1])

    Js, Jc, res = out
    from oracle.residual import optimal_error  # closed form sum_{i>k} sigma_i^2 (Eckart-Young)
    opt = optimal_error(sigma, k) if sigma is not None else None   # C4 has no closed-form spectrum
    resid = {"opt_fro": opt}
    for kind, (r, nA) in res.items():
        resid[f"{kind}_fro"] = r
        resid["normA_fro"] = nA
        resid[f"{kind}_ratio"] = r / opt if opt else None

    # roofline of the dominant kernel of the selection: the sketch (one launch per call)
    sk_ms = statistics.mean(stage_ms["sketch"])
    traffic = None
    tf = os.path.join(ROOT, "profiles", "round1", "sketch_dram_bytes.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(f"{args.config}_k{k}")
        except Exception:
            traffic = None
    if emb == "sparse_sign":
        # HBM bound: A read once + X written (Omega generated, 0 bytes), SURVEY 8(d)
        nbytes = 8.0 * (m * n + l * n)
        achieved = nbytes / (sk_ms * 1e-3) / 1e9
        peak = hbm_peak_gbs()
        roofline = {"kernel": "sk_sketch sparse sign = k_sparse_csr + k_sketch_sparse4", "bound": "hbm", "achieved": achieved, "peak": peak[0],
                    "unit": "GB/s", "frac": achieved / peak[0], "traffic": traffic, "peak_source": peak[1]}
    else:
        flops = 2.0 * l * m * n * max(1, 2 * args.piter)   # q = 0: one pass; q >= 1: 2q passes (Omega A^T, then A)
        achieved = flops / (sk_ms * 1e-3) / 1e12
        roofline = {"kernel": "sk_sketch Gaussian = k_omega_image + k_sketch_pre (+ split-K reduce)",
                    "bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS,
                    "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic,
                    "peak_source": "measured FP64 DMMA ceiling (tools/microbench/fp64_pipes.cu, "
                                   "profiles/round1/fp64_pipes.txt); MEASURED_PEAKS.json has no FP64 entry; "
                                   "cuBLAS DGEMM measured 35.5"}

    # end to end through the public API with host buffers (Algorithm 2 entry point)
    e2e = None
    if not args.no_e2e and A_np is not None and args.piter == 0:   # sk_rand_lupp has no power iterations
        A_host = torch.from_numpy(np.ascontiguousarray(A_np.T)).pin_memory().t()
        with torch.cuda.stream(stream):
            # the host-A (PCIe) path keeps speeding up for a while on a fresh box (4.6 -> 3.55 ms at
            # C2): warm it for at least W calls and one second
            t_w = time.perf_counter()
            nw = 0
            while nw < args.warmup or time.perf_counter() - t_w < 1.0:
                sk.rand_lupp(A_host, k, l, seed=seed, device=local)
                nw += 1
            times = []
            for _ in range(max(3, min(args.steps, 10))):
                e0, e1 = ev(), ev()
                e0.record(stream)
                sk.rand_lupp(A_host, k, l, seed=seed, device=local)
                e1.record(stream)
                e1.synchronize()
                times.append(e0.elapsed_time(e1))
        e2e_v = statistics.mean(times)
        if os.environ.get("SKEL_BENCH_DEBUG"):
            print("e2e times (ms):", [round(x, 3) for x in times], file=sys.stderr)
        if world > 1:
            t = torch.tensor([e2e_v], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_v = float(t[0])
        e2e = {"value": e2e_v, "unit": "ms", "h2d_bytes_per_step": int(m * n * 8), "d2h_bytes_per_step": int(k * 8),
               "api": "sk_rand_lupp (host A, pinned) -> Js on host"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and A_np is not None:
        cores, model = cpu_info()
        t0 = time.perf_counter()
        from oracle.lupp import RankError
        try:
            piv_o = oracle_selection(A_np, k, l, seed, emb, args.piter)
        except RankError as err:          # the selection is rank deficient at this k (both sides stop)
            piv_o = None
            fail_step = err.step
        cpu_ms = (time.perf_counter() - t0) * 1e3
        same = (f"{int(np.sum(piv_o == Js.cpu().numpy()))}/{k}" if piv_o is not None else
                f"n/a: oracle rank failure at step {fail_step}, GPU Js[{fail_step - 1}] = {int(Js[fail_step - 1])}")
        cpu = {"value": cpu_ms, "unit": "ms", "cores": cores, "kind": "oracle",
               "sample": f"one full {args.config} selection (sketch{' with %d power iteration(s)' % args.piter if args.piter else ''} + LUPP), numpy/BLAS on {model}",
               "pivots_equal_to_gpu": same}

    if rank == 0:
        line = {
            "metric": "skeleton-selection time (sketch+LUPP)", "value": value, "unit": "ms",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": False, "scaling": "weak" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "m": m, "n": n, "k": k, "l": l,
                       "l2": "flushed: 512 MiB overwrite between timed steps (untimed)",
                       "parallelism": "replicas" if world > 1 else "1 GPU"},
            "stages_ms": {nm: statistics.mean(v) for nm, v in stage_ms.items()},
            "sketch_rate": {"value": achieved, "unit": roofline["unit"]},
            "residual": resid,
            "cpqr_overlap": int(len(set(Js.cpu().tolist()) & set(Jc.cpu().tolist()))) if Jc is not None else None,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
