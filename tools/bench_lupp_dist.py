"""Per-step cost of the per-step-exchange column LUPP (sk_lupp_dist_*) on one GPU.

  graph+nccl  begin + k (all-gather, step) pairs captured in one CUDA graph (dist.CapturedStepwise)
              over a world-size-1 NCCL group: the real collective in the loop (a local copy at P=1,
              so this is the launch + kernel floor of the design, not its multi-GPU latency);
  kernels     the same k step kernels in a graph with the gathered records supplied by a device
              copy of P records (P = 8 emulated; decision over 8 records).
usage: python tools/bench_lupp_dist.py   (prints one line per shape)
"""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_05877_b200 as sk  # noqa: E402
from paper_2104_05877_b200.dist import CapturedStepwise  # noqa: E402

SHAPES = [("C2 k=512 (n=4096)", 4096, 512), ("C5 rank block at P=8 (nloc=8192, k=1000)", 8192, 1000),
          ("C3 cols (n=16384, k=500)", 16384, 500)]


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


def main():
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29561")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    g = torch.Generator(device="cuda").manual_seed(3)
    for name, n, k in SHAPES:
        X = torch.randn((k + 10, n), dtype=torch.float64, device="cuda", generator=g)
        cap = CapturedStepwise(X, n, k)
        ms = timed(cap.run)
        Js_ref, _, _, _ = sk.select_cols(X, k)
        same = bool((cap.sel.Js == Js_ref).all())
        # kernels only, P = 8 records per decision (7 are "none" records padding the gather)
        sel = sk.LuppDist(n, k, 0, 8, 0)
        pad = torch.full((7, sel.rec), -1.0, dtype=torch.float64, device="cuda")
        pad[:, 2] = 0.0
        gview = sel.gathered.view(8, sel.rec)

        def loop():
            sel.begin(X)
            for t in range(1, k + 1):
                gview[0].copy_(sel.cand)
                gview[1:].copy_(pad)
                sel.step(t)
        loop()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            loop()
        ms2 = timed(gr.replay)
        sel.info()
        same2 = bool((sel.Js == Js_ref).all())
        # exchange fused into the kernel (P2P mailbox, world 1): begin + k step kernels in one graph
        # (the epoch lives on the device, so the graph replays)
        box = sk.ipc_alloc(sk.mailbox_bytes(k, 1), 0)
        peers = torch.tensor([box], dtype=torch.int64, device="cuda")
        sp = sk.LuppDistP2P(n, k, 0, 1, 0, peers, box, 0)

        def ploop():
            sp.begin(X)
            for t in range(1, k + 1):
                sp.step(t)
        ploop()
        torch.cuda.synchronize()
        gp = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gp):
            ploop()
        ms3 = timed(gp.replay)
        sp.info()
        same3 = bool((sp.Js == Js_ref).all())
        sk.ipc_free(box, 0)
        ms_single = timed(lambda: sk.select_cols(X, k, want_factors=False))
        print(f"{name:42s} graph+nccl {ms:8.3f} ms ({1e3 * ms / k:6.2f} us/step, pivots==single {same})   "
              f"kernels P=8 {ms2:8.3f} ms ({1e3 * ms2 / k:6.2f} us/step, {same2})   "
              f"P2P in-kernel exchange {ms3:8.3f} ms ({1e3 * ms3 / k:6.2f} us/step, {same3})   "
              f"single-GPU cluster LUPP {ms_single:7.3f} ms", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
