#!/usr/bin/env python
"""RSA fwd+bwd throughput on B200 (BASELINE.json metric), one JSON line on rank 0.

Workload (BASELINE.json configs[1], "BERT-base 12-layer sequence-parallel
training, seq 512, batch-size scaling"): one step = the attention stack of
BERT-base -- 12 independent RSA layers (Z=12 heads, A=64, H=768) run forward
in layer order, then backward in reverse order, as in a training step --
over a synthetic batch of B = 64 sequences per GPU (global batch 64*N, the
paper's weak-scaling rule) of L = 512 tokens, the sequence
split over the N ring ranks.  value = tokens per second of the whole job
(global batch * L / step time).  Inputs are synthetic N(0,1) bf16; every
layer has its own q/k/v/dO and the per-layer working set (>1 GB) exceeds
the 126 MB L2, so no flush is needed between steps.

Arms:
  default            our sm_100a kernels (value: device-resident inputs;
                     e2e: the public ring_attention_* API with pinned host
                     buffers, H2D/D2H inside the timed region)
  --impl reference   the CPU oracle port of the reference algorithm
                     (oracle/ringseq_np.py, float64, rank-1-update matmul as
                     in ringseq/tensor_ops.py:44-72), on all host cores
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "RSA fwd+bwd tokens/s (BERT-base attention stack, 12 layers)"
UNIT = "tokens/s"
PEAKS_FILE = ROOT / "MEASURED_PEAKS.json"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=64, help="sequences per GPU")
    ap.add_argument("--seq", type=int, default=512)
    ap.add_argument("--layers", type=int, default=12)
    ap.add_argument("--heads", type=int, default=12)
    ap.add_argument("--head-size", type=int, default=64)
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of the captured step")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def config_obj(args, n):
    return {
        "workload": "BERT-base RSA stack: 12 layers x ring self-attention fwd+bwd (probs panels saved)",
        "model": "bert-base attention (Z=12, A=64, H=768)",
        "layers": args.layers,
        "global_batch": args.batch * n,
        "batch_per_gpu": args.batch,
        "seq_len": args.seq,
        "heads": args.heads,
        "head_size": args.head_size,
        "ring_ranks": n,
        "parallelism": f"seq{n}",
        "l2": "inputs larger than L2 (per-layer working set > 1 GB), no flush",
    }


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """Samples SM clock and throttle reasons via NVML every 5 ms."""

    NAMES = {
        0x1: "gpu_idle", 0x2: "applications_clocks", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clocks",
    }

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.NAMES.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.005)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join()

    def result(self):
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ------------------------------------------------------------- CPU oracle

def cpu_oracle_sample(args, threads):
    """Time the reference algorithm (oracle port) on one layer of a B=1 slice.

    Uses N_sim = threads simulated ranks on a thread pool (the reference's
    concurrent executor); returns tokens/s for the 12-layer stack.
    """
    from oracle import ringseq_np as orc

    seq, z, a = args.seq, args.heads, args.head_size
    n_sim = max(1, min(threads, 8))
    while seq % n_sim:
        n_sim -= 1
    rng = orc.make_rng(0)
    q, k, v, g = (rng.standard_normal((1, z, seq, a)) for _ in range(4))
    ch = lambda x: orc.chunks_of(x, n_sim)  # noqa: E731
    best = math.inf
    for _ in range(2):
        t0 = time.perf_counter()
        _, probs, _ = orc.ring_forward(ch(q), ch(k), ch(v), exact=True, workers=n_sim)
        orc.ring_backward(ch(q), ch(k), ch(v), probs, ch(g), exact=True, workers=n_sim)
        best = min(best, time.perf_counter() - t0)
    tokens_per_s = seq / (best * args.layers)
    sample = (f"1 RSA layer fwd+bwd, B=1 Z={z} L={seq} A={a}, {n_sim} simulated ranks on {n_sim} threads, "
              f"float64 rank-1-update matmul (oracle/ringseq_np.py exact=True); best of 2 = {best:.3f} s; "
              f"scaled to the {args.layers}-layer step")
    return tokens_per_s, n_sim, sample


def reference_arm(args):
    world, rank, _ = dist_env()
    n = max(args.gpus, world)
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    vals = []
    for _ in range(max(1, args.steps)):
        v, cores, sample = cpu_oracle_sample(args, threads)
        vals.append(v)
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": args.batch * n * args.seq / value * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_obj(args, n),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "reference is a float64 NumPy simulator; /root/reference is absent on the GPU box, so the "
                "oracle port of its algorithm (pinned bitwise to reference goldens) is timed",
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU arm

def peaks():
    try:
        return json.loads(PEAKS_FILE.read_text())
    except Exception:
        return {}


def traffic_of(kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed ncu capture."""
    try:
        t = json.loads((ROOT / "profiles" / "traffic.json").read_text())
        return t["bytes_per_launch"].get(kernel)
    except Exception:
        return None


def kernel_model(name, n, b, z, c, seq, a):
    """Algorithmic (bytes, flops) per launch of one fused kernel at one layer."""
    pe = n * b * z * c * seq  # panel elements in the launch
    ce = n * b * z * c * a    # chunk elements
    rows = n * b * z * c      # query rows
    if name == "fwd_stats":
        return 2 * 2 * ce, 2 * pe * a                 # read Q, K; S = QK^T
    if name == "fwd_probs_pv":
        return 2 * pe + 2 * 4 * ce, 4 * pe * a        # write P; read Q,K,V, write O
    if name == "fwd_resident":
        return 2 * pe + 2 * 4 * ce, 6 * pe * a        # write P; Q,K,V in, O out; QK^T twice + PV
    if name == "fwd_factored":
        return 2 * pe + 2 * 4 * ce + 4 * rows, 4 * pe * a  # write P~ and r; Q,K,V in, O out; QK^T, PV (algorithmic)
    if name == "bwd_dkdv":
        return 2 * pe + 2 * 5 * ce, 6 * pe * a        # read P; dO,Q,V in, dK,dV out; dO V^T, P^T dO, dS^T Q
    if name == "bwd_fused":
        return 2 * pe + 2 * 7 * ce, 8 * pe * a        # read P; Q,K,V,dO in, dQ,dK,dV out; dO V^T, P^T dO, dS^T Q, dS K
    if name == "bwd_dq":
        return 2 * pe + 2 * 4 * ce, 4 * pe * a        # read P; dO,K,V in, dQ out; dO V^T, dS K
    if name == "rowdot":
        return 2 * 3 * ce + 8 * rows, 3 * ce            # read dO, O, r; write D*r, dO*r
    return 0, 0


def ours(args):
    import torch

    from paper_2105_13120_b200 import engine
    from paper_2105_13120_b200.config import AttentionConfig

    world, rank, local = dist_env()
    n = max(args.gpus, world)
    if world > 1:
        from paper_2105_13120_b200 import distributed

        return distributed.bench_main(args, METRIC, UNIT, config_obj(args, world), clock_sampler=ClockSampler,
                                      peaks=peaks())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    B, Z, L, A, LAYERS = args.batch, args.heads, args.seq, args.head_size, args.layers
    c = L  # one rank per GPU: the whole sequence is this GPU's chunk at N=1
    gen = torch.Generator(device=dev).manual_seed(1234)

    def rnd():
        return torch.randn((1, B, Z, c, A), generator=gen, device=dev, dtype=torch.float32).to(torch.bfloat16)

    layers = [dict(q=rnd(), k=rnd(), v=rnd(), g=rnd()) for _ in range(LAYERS)]
    for ly in layers:
        ly["o"] = torch.empty_like(ly["q"])
        ly["p"] = torch.empty((1, B, Z, c, L), dtype=torch.bfloat16, device=dev)
        ly["r"] = torch.empty((1, B, Z, c), dtype=torch.float32, device=dev)
        ly["grads"] = (torch.empty_like(ly["q"]), torch.empty_like(ly["q"]), torch.empty_like(ly["q"]))
    dvec = torch.empty((1, B, Z, c), dtype=torch.float32, device=dev)
    g_scaled = torch.empty((1, B, Z, c, A), dtype=torch.bfloat16, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    timer = engine.KernelTimer()

    def step(tm=None):
        for ly in layers:
            engine.forward(ly["q"], ly["k"], ly["v"], path="fused", flag=flag, out=ly["o"], panel=ly["p"],
                           rowscale=ly["r"], timer=tm)
        for ly in reversed(layers):
            engine.backward(ly["q"], ly["k"], ly["v"], ly["p"], ly["g"], outputs=ly["o"], path="fused",
                            grads=ly["grads"], dvec=dvec, rowscale=ly["r"], grad_scaled=g_scaled, timer=tm)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # The whole step (every kernel of the 12 forward and 12 backward layers) captured once
    # as a CUDA graph and replayed: the same launches, without the host-side launch gaps
    run = step
    graph_used = False
    if not args.no_graph:
        try:
            graph = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream(dev)
            side.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(side):
                step()
            torch.cuda.current_stream(dev).wait_stream(side)
            with torch.cuda.graph(graph):
                step()
            graph.replay()
            torch.cuda.synchronize()
            run, graph_used = graph.replay, True
        except Exception as exc:  # capture unsupported here: time the eager launches
            print(f"cuda graph capture failed ({exc}); timing eager launches", file=sys.stderr)
            torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.steps):
            run()
        e1.record()
        torch.cuda.synchronize()
    total_ms = e0.elapsed_time(e1)
    if int(flag.item()):
        raise RuntimeError("non-finite scores in the benchmark inputs")
    ms = total_ms / args.steps
    value = B * L / (ms / 1e3)
    clocks = clk.result()

    # per-kernel timing pass: event pairs around each launch on its stream -- inside the
    # replayed graph when the step is timed as one (external events keep their timestamps
    # in a capture), else around the eager launches
    reps = max(1, min(args.steps, 3))
    tot = None
    if graph_used:
        try:
            gt = engine.KernelTimer(external=True)
            tgraph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(tgraph):
                step(gt)
            acc = {}
            for _ in range(reps):
                tgraph.replay()
                for k, (n_, ms_) in gt.totals().items():
                    c0, t0 = acc.get(k, (0, 0.0))
                    acc[k] = (c0 + n_, t0 + ms_)
            tot = acc
            timing_mode = "event pairs inside the replayed step graph"
        except Exception as exc:
            print(f"graph-captured kernel timing failed ({exc}); timing eager launches", file=sys.stderr)
            torch.cuda.synchronize()
    if tot is None:
        timer.reset()
        for _ in range(reps):
            step(timer)
        tot = timer.totals()
        timing_mode = "event pairs around eager launches"
    pk = peaks()
    hbm = pk.get("hbm_gbs", 6650.0)
    tc = pk.get("bf16_tflops_sustained", 1400.0)
    shares = {k: v[1] for k, v in tot.items()}
    dom = max(shares, key=shares.get)
    launches, dom_ms = tot[dom]
    per_launch_s = dom_ms / launches / 1e3
    byts, flops = kernel_model(dom, 1, B, Z, c, L, A)
    t_hbm, t_tc = byts / (hbm * 1e9), flops / (tc * 1e12)
    if t_hbm >= t_tc:
        roof = {"bound": "hbm", "achieved": byts / per_launch_s / 1e9, "peak": hbm, "unit": "GB/s"}
    else:
        roof = {"bound": "tensor", "achieved": flops / per_launch_s / 1e12, "peak": tc, "unit": "TFLOP/s"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["kernel"] = dom
    roof["traffic"] = traffic_of(dom)
    roof["peak_source"] = "MEASURED_PEAKS.json" if pk else "fallback (B200_PROFILING.md)"
    roof["timing"] = timing_mode
    kernels = {}
    step_kernel_ms = sum(shares.values()) / max(1, min(args.steps, 3))
    for k, (cnt, tms) in tot.items():
        b_, f_ = kernel_model(k, 1, B, Z, c, L, A)
        per = tms / cnt / 1e3
        kernels[k] = {"launches_per_step": cnt // max(1, min(args.steps, 3)), "us_per_launch": per * 1e6,
                      "share": tms / sum(shares.values()), "GB/s": b_ / per / 1e9, "TFLOP/s": f_ / per / 1e12}
    launches_per_step = sum(v["launches_per_step"] for v in kernels.values())

    # end to end through the public API, pinned host buffers
    e2e = e2e_public_api(args, dev)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic N(0,1) bf16 inputs, per-layer q/k/v/dO", "config": config_obj(args, 1),
        "launch": "cuda graph of the whole step, replayed" if graph_used else "eager launches",
        "clocks": clocks, "roofline": roof, "kernels": kernels, "kernel_ms_per_step": step_kernel_ms,
        "gpu_launches": launches_per_step * args.steps, "e2e": e2e,
    }
    if not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        v, cores, sample = cpu_oracle_sample(args, threads)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample}
    print(json.dumps(line), flush=True)


def e2e_public_api(args, dev):
    """Same step through ring_attention_forward/backward with pinned host buffers."""
    import torch

    from paper_2105_13120_b200 import AttentionConfig
    from paper_2105_13120_b200.ring_attention import ring_attention_backward, ring_attention_forward

    B, Z, L, A, LAYERS = args.batch, args.heads, args.seq, args.head_size, args.layers
    cfg = AttentionConfig(batch_size=B, seq_len=L, hidden_size=Z * A, num_heads=Z, head_size=A, num_devices=1)
    g = torch.Generator().manual_seed(99)
    host = []
    for _ in range(LAYERS):
        t = [torch.randn((B, Z, L, A), generator=g).to(torch.bfloat16).pin_memory() for _ in range(4)]
        outs = [torch.empty((B, Z, L, A), dtype=torch.bfloat16).pin_memory() for _ in range(4)]
        host.append((t, outs))
    elem = B * Z * L * A
    h2d = LAYERS * 4 * elem * 2
    d2h = LAYERS * 4 * elem * 2

    # Inputs go up on a copy stream, one step ahead: step s + 1's q/k/v/dO uploads run
    # while step s computes and copies its results down (PCIe is full duplex), into the
    # other of two device buffer sets.  Layers alternate between two compute streams; a
    # layer's forward and backward stay on its stream (the backward consumes the forward's
    # saved panel).  Every step still moves all of its inputs up and its outputs down.
    streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    copy = torch.cuda.Stream(dev)
    bufs = [[[torch.empty((B, Z, L, A), dtype=torch.bfloat16, device=dev) for _ in range(4)]
             for _ in range(LAYERS)] for _ in range(2)]
    up = [[None] * LAYERS for _ in range(2)]    # upload done, per buffer set and layer
    free = [[None] * LAYERS for _ in range(2)]  # last read of the set's layer buffers done

    def upload(set_i):
        with torch.cuda.stream(copy):
            for i, ((q, k, v, gr), _) in enumerate(host):
                if free[set_i][i] is not None:
                    copy.wait_event(free[set_i][i])
                for dst, src in zip(bufs[set_i][i], (q, k, v, gr)):
                    dst.copy_(src, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(copy)
                up[set_i][i] = ev

    def step(set_i, prefetch_next):
        saved = []
        for i, (_, outs) in enumerate(host):
            q, k, v, _ = bufs[set_i][i]
            st = streams[i % 2]
            with torch.cuda.stream(st):
                st.wait_event(up[set_i][i])
                fwd = ring_attention_forward([q], [k], [v], cfg)
                outs[0].copy_(fwd.outputs[0], non_blocking=True)
            saved.append(fwd)
        if prefetch_next:
            upload(1 - set_i)
        for i in reversed(range(LAYERS)):
            q, k, v, gr = bufs[set_i][i]
            outs = host[i][1]
            st = streams[i % 2]
            with torch.cuda.stream(st):
                bwd = ring_attention_backward([q], [k], [v], saved[i].probs, [gr], cfg)
                outs[1].copy_(bwd.grad_q[0], non_blocking=True)
                outs[2].copy_(bwd.grad_k[0], non_blocking=True)
                outs[3].copy_(bwd.grad_v[0], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(st)
                free[set_i][i] = ev

    upload(0)
    step(0, False)
    torch.cuda.synchronize()
    steps = max(1, args.e2e_steps)
    cur = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cur)
    for st in streams + [copy]:
        st.wait_event(e0)
    upload(0)  # the first timed step's inputs, inside the timed region
    for s_i in range(steps):
        step(s_i % 2, s_i + 1 < steps)
    for st in streams + [copy]:
        cur.wait_stream(st)
    e1.record(cur)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    return {"value": B * L / (ms / 1e3), "unit": UNIT, "ms_per_step": ms, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h,
            "path": "ring_attention_forward/backward (public API) on device chunks uploaded every step from "
                    "pinned host bf16 (q, k, v, dO) on a copy stream one step ahead; O, dQ, dK, dV copied to "
                    "pinned host; layers alternate over 2 compute streams"}


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
    else:
        ours(args)


if __name__ == "__main__":
    main()
