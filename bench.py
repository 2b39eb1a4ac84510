#!/usr/bin/env python
"""Benchmark of the randomized-LUPP skeleton-selection hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--k 1000] [--impl ours|reference]

Workload (default, BASELINE.json configs[4], "C5" -- the largest configuration, and the one that
fits one B200): A = U diag(i^-1.5) V^T, 131072 x 65536 FP64 (68.7 GB), U and V products of 64
Householder reflectors, built on the device from seed 1005; Gaussian Omega, k = 1000, l = 1100
(seed 2005).  One step = the C5 path of SURVEY.md section 8(d):
    S0+S1 sketch X = Omega A  ->  S2 select_cols (LUPP)  ->  S5 id_coeffs  ->  S6 residual ||A - CC^+A||_F.
value = the BASELINE.json metric "skeleton-selection time (sketch+LUPP)" = S1 + S2 device time per
step (ms, lower is better), max over ranks; ms_per_step = the whole step.  With N > 1 (torchrun)
the same matrix is column-sharded over the N GPUs (strong scaling): every rank builds
and sketches its own column block, the column LUPP exchanges per pivot step or gathers the k
LUPP-visible sketch rows once, and the residual is reduced across ranks.
--config C1..C4 run the other configurations' paths (C2 adds S2' CPQR, C3/C4 add S3 + S4).
L2 policy: a 512 MiB buffer is overwritten between timed steps (untimed); per-step CUDA events on
the library's stream.

--impl reference times the plain CPU oracle (oracle/) on the same config on the host cores (the
reference arm of this paper-only build); at C5 each step is a bounded sample
of the workload scaled to the whole selection (the sample is stated in the line).
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
    ap.add_argument("--config", default="C5")
    ap.add_argument("--k", type=int, default=None, help="default: C1 20, C2 512, C3 500, C4 200, C5 1000")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--piter", type=int, default=0,
                    help="power iterations (Rand-LUPP-qpiter, P:527): orthogonalised, eq:ortho_power_iter (P:216-224)")
    ap.add_argument("--plain-piter", action="store_true", help="the plain X = Omega (A^T A)^q of eq:def_power_iter instead")
    ap.add_argument("--dist-exchange", default="replicate", choices=["replicate", "step", "p2p"],
                    help="N > 1: column-LUPP exchange -- one k x n all-gather then replicated LUPP, one "
                         "all-gather of P records per pivot step (CUDA graph), or the records stored into "
                         "the peers' mailboxes by the step kernel itself (NVLink peer memory, CUDA graph)")
    ap.add_argument("--sketch-tuning", default="",
                    help="path,bm,splits,chunk[,warps] for sk_set_sketch_tuning (A/B of the dense sketch's plans)")
    return ap.parse_args()


def workload(args):
    from inputs import CONFIGS
    cfg = CONFIGS[args.config]
    if args.k is None:
        args.k = {"C1": 20, "C2": 512, "C3": 500, "C4": 200, "C5": 1000}[args.config]
        if getattr(args, "piter", 0) and args.config == "C2" and getattr(args, "plain_piter", False):
            # the PLAIN X = Omega (A^T A)^q squares the C2 spectrum (10^(-i/25)): beyond k ~ 390 the
            # sketch is rank deficient at LUPP's 1e-14 threshold (both the oracle and the GPU stop there);
            # the orthogonalised iteration (the default) runs at k = 512
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
        desc += (f", {args.piter} plain power iteration(s) X = Omega (A^T A)^q (Rand-LUPP-{args.piter}piter)"
                 if getattr(args, "plain_piter", False) else
                 f", {args.piter} orthogonalised power iteration(s) X = ortho(Y_q)^T A (eq:ortho_power_iter, "
                 f"Rand-LUPP-{args.piter}piter)")
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


def oracle_selection(A, k, l, seed, emb="gaussian", piter=0, plain=False):
    """The oracle's sketch (with q = piter power iterations, orthogonalised unless plain) + LUPP
    (test infrastructure; timed as the CPU baseline)."""
    from oracle import lupp as o_lupp
    from oracle import sketch as o_sketch
    if piter == 0:
        X = o_sketch.sketch(A, l, emb, seed)
    elif plain:
        X = o_sketch.sketch_power(A, l, emb, seed, piter)
    else:
        X = o_sketch.sketch_power_ortho(A, l, emb, seed, piter)
    piv, _, _, _ = o_lupp.select_cols(X, k)
    return piv


C5_SAMPLE_COLS = 1024


def c5_oracle_sample(get_block, m, n, k, l, seed):
    """The oracle on a bounded sample of C5's selection, scaled to the whole selection (ms):
    the full Gamma (l x m) generated as the oracle does it, the sketch of C5_SAMPLE_COLS columns of
    A (X = Gamma A is column-separable, so the whole sketch costs n / C5_SAMPLE_COLS times that), and
    the oracle's LUPP on a seeded n x k Gaussian panel of C5's panel shape (the LUPP's work does not
    depend on the values).  Returns (value_ms, parts, X block) -- test infrastructure on the host."""
    from oracle import lupp as o_lupp
    from oracle import omega as o_omega
    Ab = np.asarray(get_block(0, C5_SAMPLE_COLS), dtype=np.float64)
    t0 = time.perf_counter()
    G = o_omega.gaussian(seed, l, m)
    t1 = time.perf_counter()
    Xb = G @ Ab
    t2 = time.perf_counter()
    del G
    P = np.random.default_rng(7).standard_normal((k, n))
    t3 = time.perf_counter()
    o_lupp.select_cols(P, k, fast=True)
    t4 = time.perf_counter()
    parts = {"gamma_gen_ms": (t1 - t0) * 1e3, "sketch_ms": (t2 - t1) * 1e3 * n / C5_SAMPLE_COLS,
             "lupp_ms": (t4 - t3) * 1e3}
    return sum(parts.values()), parts, Xb


def c5_sample_desc(model):
    return (f"C5 oracle sample scaled to the whole selection: full Gamma generation (numpy Philox), sketch of "
            f"{C5_SAMPLE_COLS} of 65536 columns x 64, plain-C oracle LUPP on a 65536 x 1000 seeded panel; on {model}")


def c5_e2e(args, sk, A, m, n, k, l, seed, local, stream, ev, Js_dev):
    """e2e at C5 through the public Algorithm-2 call sk_rand_lupp with A in pinned HOST memory
    (68.7 GB, page-locked with cudaHostRegister): every call copies all of A host -> device in
    column blocks (a 3-slot device ring, copy of block b overlapping the sketch of block b - 1)
    and returns J_s on the host."""
    import torch
    Ah = np.empty((n, m), dtype=np.float64)                       # rows = columns of A
    cudart = torch.cuda.cudart()
    reg = cudart.cudaHostRegister(Ah.ctypes.data, Ah.nbytes, 0)
    if int(reg) != 0:
        return {"value": None, "unit": "ms", "error": f"cudaHostRegister failed ({int(reg)})"}
    try:
        Aht = torch.from_numpy(Ah)
        At = A.t()
        for j0 in range(0, n, 4096):                                 # device -> registered host, untimed
            Aht[j0:j0 + 4096].copy_(At[j0:j0 + 4096])
        torch.cuda.synchronize()
        A_host = Aht.t()
        times = []
        with torch.cuda.stream(stream):
            for it in range(max(1, min(args.warmup, 2)) + max(2, min(args.steps, 5))):
                e0, e1 = ev(), ev()
                e0.record(stream)
                Jh, _ = sk.rand_lupp(A_host, k, l, seed=seed, device=local)
                e1.record(stream)
                e1.synchronize()
                if it >= max(1, min(args.warmup, 2)):
                    times.append(e0.elapsed_time(e1))
        same = int(np.sum(np.asarray(Jh) == Js_dev.cpu().numpy()))
        return {"value": statistics.mean(times), "unit": "ms", "h2d_bytes_per_step": int(m * n * 8),
                "d2h_bytes_per_step": int(k * 8), "api": "sk_rand_lupp (host A, page-locked) -> Js on host",
                "pivots_equal_to_device_path": f"{same}/{k}"}
    finally:
        cudart.cudaHostUnregister(Ah.ctypes.data)
        del Ah


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


def lupp_report(ms, rows, k):
    """SURVEY 8(d) figures of one LUPP call: rows x k panel, k pivot steps."""
    flops, nbytes = float(rows) * k * k, 16.0 * rows * k
    t_lb = max(flops / (FP64_PEAK_TFLOPS * 1e12), nbytes / (hbm_peak_gbs()[0] * 1e9)) * 1e3
    return {"ms": ms, "us_per_step": ms * 1e3 / k, "gbs": nbytes / (ms * 1e-3) / 1e9,
            "tflops": flops / (ms * 1e-3) / 1e12, "bound_ms": t_lb, "frac_of_bound": t_lb / ms,
            "bound": "k sequential argmaxes (chain); bandwidth / flop bound max(F/P64, B/BW) as frac_of_bound"}


def run_reference(args):
    """--impl reference: the oracle on the host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg, k, l, seed, desc = workload(args)
    if args.config == "C5":   # 68.7 GB does not fit the host oracle: a bounded sample per step (stated)
        from inputs import c5 as c5in
        m, n = c5in.M5, c5in.N5
        cores, model = cpu_info()
        steps = max(1, min(args.steps, 3))
        warm = min(args.warmup, 1)
        times = []
        for it in range(warm + steps):
            v, parts, _ = c5_oracle_sample(lambda a, b: c5in.build_block_host(a, b), m, n, k, l, seed)
            if it >= warm:
                times.append(v)
        v = statistics.mean(times)
        line = {
            "impl": "reference", "metric": "skeleton-selection time (sketch+LUPP)", "value": v, "unit": "ms",
            "n_gpus": args.gpus, "steps": steps, "warmup": warm, "ms_per_step": v, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "m": m, "n": n, "k": k, "l": l},
            "cpu_baseline": {"value": v, "unit": "ms", "cores": cores, "kind": "oracle", "sample": c5_sample_desc(model),
                             "parts_ms": parts},
            "e2e": {"value": v, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)
        return 0
    A, _ = make_input(args, cfg)
    cores, model = cpu_info()
    steps = max(1, min(args.steps, 3))
    warm = min(args.warmup, 1)
    for _ in range(warm):
        oracle_selection(A, k, l, seed, cfg["emb"], args.piter, args.plain_piter)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        oracle_selection(A, k, l, seed, cfg["emb"], args.piter, args.plain_piter)
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


def apply_sketch_tuning(args, sk, device):
    if args.sketch_tuning:
        t = [int(x) for x in args.sketch_tuning.split(",")]
        sk.set_sketch_tuning(*t[:4], warps=t[4] if len(t) > 4 else 0, device=device)


def main_dist(args, world, rank, local):
    """N > 1 GPUs (torchrun): the column-sharded path of SURVEY 8(e) on the same C5 matrix
    (strong scaling: rank r builds and holds only its contiguous block of A's 65536 columns, built
    on its device from the same seed).  The library's distributed context (sk_create_dist, one
    NCCL communicator owned by the library) does every exchange.  One step = sketch of the local
    block (Gamma regenerated from the seed, no communication) -> column LUPP (exchange
    "replicate": one all-gather of the k LUPP-visible sketch rows, then the cluster LUPP on
    identical bytes; "step": one all-gather of P candidate records per pivot step, CUDA graph) ->
    ID coefficients of the local columns -> column-ID residual (C by one all-gather, Q_C by
    Cholesky QR over row blocks with k x k all-reduces, one all-reduce of the squared sums).
    value = sketch + selection time, max over ranks."""
    import torch
    import torch.distributed as dist

    import paper_2104_05877_b200 as sk
    from paper_2104_05877_b200.dist import shard

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.Stream(dev)
    cfg, k, l, seed, desc = workload(args)
    if args.config != "C5":
        raise SystemExit("the multi-GPU bench runs the column-sharded C5 workload (--config C5)")
    from inputs import c5 as c5in
    m, n = c5in.M5, c5in.N5
    col0, ncols = shard(n, world, rank)
    with torch.cuda.stream(stream):
        A, sigma = c5in.build_on_device(dev, col0=col0, ncols=ncols)
        flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
        Xbuf = torch.empty((l, ncols), dtype=torch.float64, device=dev)
    torch.cuda.synchronize(dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    exchange = "step" if args.dist_exchange == "step" else "replicate"
    with torch.cuda.stream(stream):
        sess = sk.DistSession(n, None, local, exchange)

    def step(record):
        e = [ev() for _ in range(5)]
        e[0].record(stream)
        X = sk.sketch(A, l, "gaussian", seed, out=Xbuf)
        e[1].record(stream)
        Js, Lf, _, _ = sk.select_cols(X, k, check=False)
        e[2].record(stream)
        Z, _ = sk.id_coeffs(Lf, Js)
        e[3].record(stream)
        r, nA = sk.residual(A, Js, None, "col_id")
        e[4].record(stream)
        record(e)
        return Js, r, nA

    with torch.cuda.stream(stream), sess:
        apply_sketch_tuning(args, sk, local)                 # on the distributed context
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
        e2e = None
        if not args.no_e2e:   # sk_rand_lupp on the distributed context, each rank's block in host memory
            e2e = c5_e2e(args, sk, A, m, ncols, k, l, seed, local, stream, ev, out[0])
            v = torch.tensor([e2e["value"] if e2e.get("value") is not None else float("nan")], dtype=torch.float64,
                             device=dev)
            dist.all_reduce(v, op=dist.ReduceOp.MAX)
            e2e["value"] = float(v[0])
            e2e["h2d_bytes_per_step"] = int(m * n * 8)
            e2e["api"] += f" on the column-sharded context, {world} ranks (host block per rank), max over ranks"
    sess.close()
    sk_ms = statistics.mean(e[0].elapsed_time(e[1]) for e in recs)
    sel_ms = statistics.mean(e[0].elapsed_time(e[2]) for e in recs)
    step_ms = statistics.mean(e[0].elapsed_time(e[4]) for e in recs)
    stage = {"sketch": sk_ms, "select_cols_lupp": statistics.mean(e[1].elapsed_time(e[2]) for e in recs),
             "id_coeffs": statistics.mean(e[2].elapsed_time(e[3]) for e in recs),
             "residual": statistics.mean(e[3].elapsed_time(e[4]) for e in recs)}
    t = torch.tensor([sel_ms, step_ms, sk_ms] + list(stage.values()), dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    sel_ms, step_ms, sk_ms_max = float(t[0]), float(t[1]), float(t[2])
    stage = dict(zip(stage, [float(x) for x in t[3:]]))
    Js, r, nA = out
    achieved = 2.0 * l * m * ncols / (sk_ms * 1e-3) / 1e12
    if rank == 0:
        from oracle.residual import optimal_error
        opt = optimal_error(sigma, k)
        line = {
            "metric": "skeleton-selection time (sketch+LUPP)", "value": sel_ms, "unit": "ms",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc + f", column-sharded over {world} GPUs", "m": m, "n": n, "k": k, "l": l,
                       "parallelism": f"column-sharded x{world}", "lupp_exchange": exchange,
                       "l2": "flushed: 512 MiB overwrite between timed steps (untimed); A (68.7 GB) >> L2"},
            "stages_ms": stage,
            "lupp": {"select_cols": lupp_report(stage["select_cols_lupp"], n, k)},
            "residual": {"col_id_fro": r, "normA_fro": nA, "opt_fro": opt, "col_id_ratio": r / opt},
            "roofline": {"kernel": "sk_sketch Gaussian (k_omega_image + k_sketch_pre per K-chunk), rank 0's block",
                         "bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS,
                         "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS, "traffic": None},
            "cpu_baseline": None,
            "e2e": e2e,
            "gpu_launches": int(launches), "clocks": clk.summary(),
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
    apply_sketch_tuning(args, sk, local)                     # A/B only; the default line leaves the planner alone

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
             else sk.sketch_power(A, l, emb, seed, args.piter, cfg.get("zeta", 8), ortho=not args.plain_piter))
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
        return Js, Jc, res, X

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

    Js, Jc, res, X_last = out
    from oracle.residual import optimal_error  # closed form sum_{i>k} sigma_i^2 (Eckart-Young)
    opt = optimal_error(sigma, k) if sigma is not None else None   # C4 has no closed-form spectrum
    resid = {"opt_fro": opt}
    for kind, (r, nA) in res.items():
        resid[f"{kind}_fro"] = r
        resid["normA_fro"] = nA
        resid[f"{kind}_ratio"] = r / opt if opt else None

    # roofline of the dominant kernel of the selection: the sketch (one launch per call)
    sk_ms = statistics.mean(stage_ms["sketch"])
    traffic = traffic_note = None
    tf = os.path.join(ROOT, "profiles", "round2", "sketch_dram_bytes.json")
    if os.path.exists(tf):
        try:
            # measured for the one-pass sketch only (tools/sketch_traffic.py); power iterations differ
            tj = json.load(open(tf))
            traffic = None if args.piter else tj.get(f"{args.config}_k{k}")
            traffic_note = tj.get("_note") if traffic is not None else None
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
    roofline["algorithmic_bytes"] = 8.0 * (m * n + l * n)
    roofline["traffic_note"] = traffic_note

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
    elif not args.no_e2e and args.config == "C5" and args.piter == 0:
        e2e = c5_e2e(args, sk, A, m, n, k, l, seed, local, stream, ev, Js)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.config == "C5":
        cores, model = cpu_info()
        At = A.t()
        v, parts, Xb = c5_oracle_sample(lambda a, b: At[a:b].cpu().numpy().T, m, n, k, l, seed)
        xg = X_last[:, :C5_SAMPLE_COLS].cpu().numpy()
        cpu = {"value": v, "unit": "ms", "cores": cores, "kind": "oracle", "sample": c5_sample_desc(model),
               "parts_ms": parts,
               "sample_check": f"oracle X(:, 0:{C5_SAMPLE_COLS}) vs GPU: rel. Frobenius "
                               f"{float(np.linalg.norm(xg - Xb) / np.linalg.norm(Xb)):.2e}"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline and A_np is not None:
        cores, model = cpu_info()
        t0 = time.perf_counter()
        from oracle.lupp import RankError
        try:
            piv_o = oracle_selection(A_np, k, l, seed, emb, args.piter, args.plain_piter)
        except RankError as err:          # the selection is rank deficient at this k (both sides stop)
            piv_o = None
            fail_step = err.step
        cpu_ms = (time.perf_counter() - t0) * 1e3
        same = (f"{int(np.sum(piv_o == Js.cpu().numpy()))}/{k}" if piv_o is not None else
                f"n/a: oracle rank failure at step {fail_step}, GPU Js[{fail_step - 1}] = {int(Js[fail_step - 1])}")
        cpu = {"value": cpu_ms, "unit": "ms", "cores": cores, "kind": "oracle",
               "sample": f"one full {args.config} selection (sketch{' with %d power iteration(s)' % args.piter if args.piter else ''} + LUPP), numpy/BLAS on {model}",
               "pivots_equal_to_gpu": same}
        if args.config in ("C1", "C2"):   # the small configs also at one thread
            from threadpoolctl import threadpool_limits
            with threadpool_limits(limits=1):
                t0 = time.perf_counter()
                try:
                    oracle_selection(A_np, k, l, seed, emb, args.piter, args.plain_piter)
                except RankError:
                    pass
                cpu["value_1thread"] = (time.perf_counter() - t0) * 1e3

    # every LUPP against max(F / P64, B / BW) with F = rows * k^2 flop and B = 16 * rows * k
    # bytes (the panel read and the factor written once); the k sequential argmaxes bound it in practice
    lupp = {"select_cols": lupp_report(statistics.mean(stage_ms["select_cols_lupp"]), n, k)}
    if do_rows:
        lupp["select_rows"] = lupp_report(statistics.mean(stage_ms["select_rows_lupp"]), m, k)

    if rank == 0:
        line = {
            "metric": "skeleton-selection time (sketch+LUPP)", "value": value, "unit": "ms",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": False, "scaling": "strong" if args.config == "C5" else "weak",   # C5: the same matrix column-sharded at N > 1
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "m": m, "n": n, "k": k, "l": l,
                       "l2": "flushed: 512 MiB overwrite between timed steps (untimed)",
                       "parallelism": "replicas" if world > 1 else "1 GPU"},
            "stages_ms": {nm: statistics.mean(v) for nm, v in stage_ms.items()},
            "stages_median_ms": {nm: statistics.median(v) for nm, v in stage_ms.items()},
            "sketch_rate": {"value": achieved, "unit": roofline["unit"]},
            "lupp": lupp,
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
