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
    ap.add_argument("--e2e-steps", type=int, default=16)
    ap.add_argument("--e2e-checks", default="deferred", choices=["sync", "deferred"],
                    help="RSA_B200_CHECK for the e2e leg: deferred reads each forward's status flag at its "
                         "backward instead of a host sync per forward call")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of the captured step")
    ap.add_argument("--ring-ranks", type=int, default=1,
                    help="N=1 only: split the sequence over this many logical ring ranks resident on the GPU "
                         "(config 1 = --ring-ranks 4 --batch 4 --layers 1)")
    ap.add_argument("--attn", default="panel", choices=["panel", "stream"],
                    help="panel: the reference's saved probability panels; stream: O(L) state, P recomputed")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def config_obj(args, n):
    return {
        "workload": ("BERT-base RSA stack: 12 layers x ring self-attention fwd+bwd (probs panels saved)"
                     if args.attn == "panel" else
                     "BERT-base RSA stack: 12 layers x ring self-attention fwd+bwd, stream mode (row statistics "
                     "saved, probabilities recomputed in the backward)"),
        "attn": args.attn,
        "model": "bert-base attention (Z=12, A=64, H=768)",
        "layers": args.layers,
        "global_batch": args.batch * n,
        "batch_per_gpu": args.batch,
        "seq_len": args.seq,
        "heads": args.heads,
        "head_size": args.head_size,
        "ring_ranks": n if n > 1 else args.ring_ranks,
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

def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


def _oracle_layer(args, n_sim, workers, rng):
    """One RSA layer fwd+bwd of ONE sequence (B=1, Z, L, A) through the oracle port of the
    reference algorithm (oracle/ringseq_np.py, exact=True: float64 rank-1-update matmul as
    ringseq/tensor_ops.py:44-72) with n_sim simulated ring ranks on `workers` threads."""
    from oracle import ringseq_np as orc

    q, k, v, g = (rng.standard_normal((1, args.heads, args.seq, args.head_size)) for _ in range(4))
    ch = lambda x: orc.chunks_of(x, n_sim)  # noqa: E731
    t0 = time.perf_counter()
    _, probs, _ = orc.ring_forward(ch(q), ch(k), ch(v), exact=True, workers=workers)
    orc.ring_backward(ch(q), ch(k), ch(v), probs, ch(g), exact=True, workers=workers)
    return time.perf_counter() - t0


def _sim_ranks(args, threads):
    n_sim = max(1, min(threads, 8))
    while args.seq % n_sim:
        n_sim -= 1
    return n_sim


def cpu_oracle_sample(args, threads):
    """cpu_baseline of our arm: one layer of one sequence (bounded, ~0.3 s on 8 cores),
    best of 2, as tokens/s of the layer stack (per-token work is batch-independent)."""
    from oracle import ringseq_np as orc

    n_sim = _sim_ranks(args, threads)
    rng = orc.make_rng(0)
    best = min(_oracle_layer(args, n_sim, n_sim, rng) for _ in range(2))
    tokens_per_s = args.seq / (best * args.layers)
    sample = (f"1 RSA layer fwd+bwd of 1 sequence (B=1 Z={args.heads} L={args.seq} A={args.head_size}), "
              f"{n_sim} simulated ranks on {n_sim} threads, float64 rank-1-update matmul (oracle/ringseq_np.py "
              f"exact=True); best of 2 = {best:.3f} s per layer; tokens/s = L / ({args.layers} x layer time)")
    return tokens_per_s, n_sim, sample


def reference_arm(args):
    """--impl reference: the reference's CPU algorithm on the host cores, timed per step.

    /root/reference does not travel to the GPU box, so the oracle port (pinned bitwise to
    goldens generated from the unmodified reference) is what runs.  One step is a bounded
    sample of the workload: ONE of the B sequences through all `layers` RSA layers fwd+bwd
    (the same work per token as the GPU step), with the sequence split over simulated ring
    ranks run on all host threads (the reference's concurrent executor).  `ms_per_step` and
    `steps` are what actually ran; `value` = tokens of the sample / step time.
    """
    world, rank, _ = dist_env()
    n = max(args.gpus, world)
    if rank != 0:
        return
    from oracle import ringseq_np as orc

    threads = host_threads()
    n_sim = _sim_ranks(args, threads)
    rng = orc.make_rng(0)

    def one_step():
        return sum(_oracle_layer(args, n_sim, n_sim, rng) for _ in range(args.layers))

    warm = min(args.warmup, 1)
    for _ in range(warm):
        one_step()
    times = [one_step() for _ in range(max(1, args.steps))]
    ms = 1e3 * sum(times) / len(times)
    value = args.seq / (ms / 1e3)
    seq_one = _oracle_layer(args, n_sim, 1, rng)  # the sequential executor: one core
    sample = (f"per step: 1 of the {args.batch * n} sequences (B=1 Z={args.heads} L={args.seq} A={args.head_size}) "
              f"through all {args.layers} layers fwd+bwd, {n_sim} simulated ring ranks on {n_sim} threads, float64 "
              f"rank-1-update matmul (oracle/ringseq_np.py exact=True)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n,
        "steps": len(times), "warmup": warm, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic N(0,1) float64 (make_rng(0))", "config": config_obj(args, n),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": n_sim, "kind": "port", "sample": sample,
                         "cpu_model": cpu_model(), "cpu_count": os.cpu_count(), "affinity": threads,
                         "sequential_executor": {"value": args.seq / (seq_one * args.layers), "unit": UNIT,
                                                 "cores": 1, "layer_s": seq_one}},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "step_sample": {"sequences_per_step": 1, "of_global_batch": args.batch * n, "layers": args.layers,
                        "step_times_s": [round(t, 4) for t in times]},
        "note": "reference is a float64 NumPy simulator; /root/reference is absent on the GPU box, so the "
                "oracle port of its algorithm (pinned bitwise to reference goldens) is timed; warm-up capped at "
                "1 step (no device state to warm)",
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
    if name == "bwd_panel_fused":  # one panel read at any length; dQ partials through L2 (not algorithmic)
        return 2 * pe + 2 * 7 * ce, 8 * pe * a
    if name == "bwd_dkdv_dq":  # the pair as one backward: the panel read twice (algorithmic: once)
        return 2 * pe + 2 * 7 * ce, 8 * pe * a
    if name == "rowdot":
        return 2 * 3 * ce + 8 * rows, 3 * ce            # read dO, O, r; write D*r, dO*r
    if name == "fwd_stream":
        return 2 * 4 * ce + 8 * rows, 4 * pe * a        # Q,K,V in, O out, r and m out; QK^T, PV (algorithmic)
    if name == "bwd_stream":
        return 2 * 7 * ce + 8 * rows, 8 * pe * a        # Q,K,V,dO' in, dQ,dK,dV out, m, D' in; the 4 bwd products
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
    R = args.ring_ranks  # logical ring ranks resident on this GPU (1: the whole sequence is one chunk)
    if L % R:
        raise SystemExit(f"seq {L} not divisible by {R} ring ranks")
    c = L // R
    gen = torch.Generator(device=dev).manual_seed(1234)

    def rnd():
        return torch.randn((R, B, Z, c, A), generator=gen, device=dev, dtype=torch.float32).to(torch.bfloat16)

    layers = [dict(q=rnd(), k=rnd(), v=rnd(), g=rnd()) for _ in range(LAYERS)]
    stream = args.attn == "stream"
    for ly in layers:
        ly["o"] = torch.empty_like(ly["q"])
        if stream:  # the stream mode saves two fp32 numbers per row instead of the (c x L) panel
            ly["m"] = torch.empty((R, B, Z, c), dtype=torch.float32, device=dev)
            ly["dq_acc"] = torch.empty((R, B, Z, c, A), dtype=torch.float32, device=dev)
        else:
            ly["p"] = torch.empty((R, B, Z, c, L), dtype=torch.bfloat16, device=dev)
            if engine.backward_kind(R, B, Z, c, A) == "bwd_panel_fused":  # its dQ accumulator
                ly["dq_acc"] = torch.empty((R, B, Z, c, A), dtype=torch.float32, device=dev)
        ly["r"] = torch.empty((R, B, Z, c), dtype=torch.float32, device=dev)
        ly["grads"] = (torch.empty_like(ly["q"]), torch.empty_like(ly["q"]), torch.empty_like(ly["q"]))
    dvec = torch.empty((R, B, Z, c), dtype=torch.float32, device=dev)
    g_scaled = torch.empty((R, B, Z, c, A), dtype=torch.bfloat16, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)

    def fwd_layer(ly):
        if stream:
            engine.forward_stream(ly["q"], ly["k"], ly["v"], flag=flag, out=ly["o"], rowscale=ly["r"], rowmax=ly["m"])
        else:
            engine.forward(ly["q"], ly["k"], ly["v"], path="fused", flag=flag, out=ly["o"], panel=ly["p"],
                           rowscale=ly["r"])

    def bwd_layer(ly, prologue=True):
        if stream:
            from paper_2105_13120_b200 import tensor_ops as ops_

            if prologue:
                ops_.rowdot_scale(ly["g"], ly["o"], ly["r"], out=dvec, a_scaled=g_scaled)
            return engine.stream_backward_kernels(ly["q"], ly["k"], ly["v"], g_scaled, ly["m"], dvec, ly["grads"],
                                                  dq_acc=ly["dq_acc"])
        engine.backward(ly["q"], ly["k"], ly["v"], ly["p"], ly["g"], outputs=ly["o"], path="fused",
                        grads=ly["grads"], dvec=dvec, rowscale=ly["r"], grad_scaled=g_scaled, prologue=prologue,
                        dq_acc=ly.get("dq_acc"))

    def step():
        for ly in layers:
            fwd_layer(ly)
        for ly in reversed(layers):
            bwd_layer(ly)

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

    # Per-kernel timing: one CUDA graph per kernel type holding only that type's launches
    # of the step (the step's own arguments, in step order), replayed and timed with an
    # event pair on the capture/replay stream.  No timing node sits inside a measured graph,
    # so the per-type times add up to the step time (up to launch-gap noise) and the
    # dominant kernel's per-launch time is its own.
    from paper_2105_13120_b200 import tensor_ops as ops

    def launches(kind):
        def run_kind():
            if kind in ("fwd_factored", "fwd_stream"):
                for ly in layers:
                    fwd_layer(ly)
            elif kind == "rowdot":
                for ly in reversed(layers):
                    ops.rowdot_scale(ly["g"], ly["o"], ly["r"], out=dvec, a_scaled=g_scaled)
            else:
                for ly in reversed(layers):
                    bwd_layer(ly, prologue=False)
        return run_kind

    reps = max(3, min(args.steps, 10))
    bwd_kind = engine.backward_kind(R, B, Z, c, A)
    kinds = ["fwd_stream", "rowdot", "bwd_stream"] if stream else ["fwd_factored", "rowdot", bwd_kind]
    replays = {}
    for kind in kinds:
        fn = launches(kind)
        fn()
        torch.cuda.synchronize()
        replays[kind] = fn
        if graph_used:
            kg = torch.cuda.CUDAGraph()
            with torch.cuda.graph(kg):
                fn()
            replays[kind] = kg.replay
            kg.replay()
    replays["step"] = run
    torch.cuda.synchronize()
    # interleaved rounds: the step graph, then each type's graph, each replayed `reps` times
    # back to back under one event pair (steady state, like the timed loop), so clock drift
    # affects every figure alike and the per-type times add up to the step
    rounds = 3
    acc = {k: 0.0 for k in replays}
    with ClockSampler(local) as kclk:
        for _ in range(rounds):
            for kind, replay in replays.items():
                # an idle gap before each segment, so every segment (like the headline's timed
                # loop) starts from the same thermal / power state instead of a power-capped one
                time.sleep(0.25)
                k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                k0.record()
                for _ in range(reps):
                    replay()
                k1.record()
                torch.cuda.synchronize()
                acc[kind] += k0.elapsed_time(k1)
    type_ms = {k: acc[k] / (rounds * reps) for k in kinds}
    step_ref_ms = acc["step"] / (rounds * reps)
    kernel_clocks = kclk.result()
    timing_mode = (f"per kernel type: a CUDA graph of that type's {LAYERS} launches of the step, replayed {reps}x back "
                   f"to back per segment after a 0.25 s idle gap, {rounds} rounds interleaved with the step graph; "
                   f"event pair on the replay stream")
    pk = peaks()
    hbm = pk.get("hbm_gbs", 6650.0)
    tc = pk.get("bf16_tflops_sustained", 1400.0)
    dom = max(type_ms, key=type_ms.get)
    per_launch_s = type_ms[dom] / LAYERS / 1e3
    byts, flops = kernel_model(dom, R, B, Z, c, L, A)
    t_hbm, t_tc = byts / (hbm * 1e9), flops / (tc * 1e12)
    if t_hbm >= t_tc:
        roof = {"bound": "hbm", "achieved": byts / per_launch_s / 1e9, "peak": hbm, "unit": "GB/s"}
    else:
        roof = {"bound": "tensor", "achieved": flops / per_launch_s / 1e12, "peak": tc, "unit": "TFLOP/s"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["kernel"] = dom
    roof["us_per_launch"] = per_launch_s * 1e6
    roof["algorithmic_bytes_per_launch"] = byts
    roof["traffic"] = traffic_of(dom)
    roof["traffic_source"] = "profiles/traffic.json (ncu --set full capture of this kernel at this shape)"
    roof["peak_source"] = "MEASURED_PEAKS.json" if pk else "fallback (B200_PROFILING.md)"
    roof["timing"] = timing_mode
    # whole step against SURVEY.md section 8(d): 4*P_e + 16*C_e algorithmic HBM bytes per layer
    p_e, c_e = R * B * Z * c * L, R * B * Z * c * A  # every resident rank's panel and chunks
    step_bytes = LAYERS * (4 * p_e + 16 * c_e)
    roof["step"] = {"bytes": step_bytes, "achieved": step_bytes / (ms / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                    "frac": step_bytes / (ms / 1e3) / 1e9 / hbm,
                    "definition": "SURVEY.md 8(d): per layer 4*P_e (bf16 panel written + read) + 16*C_e "
                                  "(q, k, v, o, dO, dQ, dK, dV bf16)"}
    kernels = {}
    for k, tms in type_ms.items():
        b_, f_ = kernel_model(k, R, B, Z, c, L, A)
        per = tms / LAYERS / 1e3
        kernels[k] = {"launches_per_step": LAYERS, "us_per_launch": per * 1e6, "ms_per_step": tms,
                      "share_of_step": tms / step_ref_ms, "GB/s": b_ / per / 1e9, "TFLOP/s": f_ / per / 1e12}
    kernel_sum = sum(type_ms.values())
    # fwd + rowdot + one backward launch, or two for the two-kernel backward and the stream
    # backward (rsa_bwd_stream_fused + dQ's bf16 cast, or the deterministic kv + q pair)
    launches_per_step = LAYERS * (4 if (stream or bwd_kind != "bwd_fused") else 3)

    # parity of the timed path: re-run one step, then check sampled heads of the first and
    # last layer against the float64 oracle (ringseq/reference.py:66-103 per head)
    run()
    torch.cuda.synchronize()
    parity = sampled_parity(layers, B, Z, seed=11)

    # end to end through the public API, pinned host buffers
    e2e = e2e_public_api(args, dev)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic N(0,1) bf16 inputs, per-layer q/k/v/dO", "config": config_obj(args, 1),
        "launch": "cuda graph of the whole step, replayed" if graph_used else "eager launches",
        "clocks": clocks, "roofline": roof, "kernels": kernels, "kernel_ms_sum": kernel_sum,
        "kernel_sum_over_step": kernel_sum / step_ref_ms, "step_ms_interleaved": step_ref_ms,
        "kernel_timing_clocks": kernel_clocks, "gpu_launches": launches_per_step * args.steps, "e2e": e2e,
        "parity": parity, "max_seq_len": max_seq_len(args, torch.cuda.mem_get_info(dev)[1]),
    }
    if not args.no_cpu_baseline:
        v, cores, sample = cpu_oracle_sample(args, host_threads())
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample}
    print(json.dumps(line), flush=True)


def max_seq_len(args, total_hbm):
    """The metric's second half, "max seq length per box", for BASELINE config 3's workload
    (BERT-base attention stack, B = 4, 12 layers, every layer's state saved), DERIVED from
    the state each mode keeps per token against this GPU's HBM (the sweep that measures it
    and the proof run at the stream maximum are tools/stream_sweep.py's, in
    profiles/r2s3_stream_sweep.json: 536,576 tokens run, 12,288 for panels).  Per layer and
    token: q, k, v, O (4 x Z*A bf16) plus, stream mode, m and r (2 x Z fp32) or, panel
    mode, its row of the (c x L) panel (Z*L bf16); the backward adds one layer's transient
    gradient buffers (dQ fp32 accumulator, dO, dO*r, dQ/dK/dV, D).  Max L grows linearly
    with N in stream mode (state O(L/N) per GPU) and as sqrt(N) with panels."""
    Z, A, layers, B = args.heads, args.head_size, args.layers, 4
    per_tok = layers * (4 * Z * A * 2) + (Z * A * 4 + 5 * Z * A * 2 + Z * 4)  # + one layer's backward transients
    stream = (layers * 2 * Z * 4 + per_tok) * B
    budget = 0.97 * total_hbm
    l_stream = int(budget // stream) // 4096 * 4096
    # panel: B * (per_tok + layers * Z * 2 * L) * L <= budget
    a_, b_ = B * layers * Z * 2, B * per_tok
    l_panel = int((-b_ + (b_ * b_ + 4 * a_ * budget) ** 0.5) / (2 * a_)) // 1024 * 1024
    return {"stream": l_stream, "panel": l_panel, "batch": B, "layers": layers, "method": "derived (bytes per token "
            "against this GPU's HBM); measured: profiles/r2s3_stream_sweep.json", "stream_per_8_gpus_derived": 8 * l_stream,
            "panel_per_8_gpus_derived": int(l_panel * 8 ** 0.5)}


def sampled_parity(layers, B, Z, seed, heads_per_layer=8):
    """Max errors of sampled heads of the first and last layer of the timed step vs the
    oracle (oracle.attention_head_sampled, float64), with the parity tests' gates."""
    import numpy as np
    import torch

    from oracle import ringseq_np as orc
    from paper_2105_13120_b200 import engine

    rng = np.random.default_rng(seed)
    worst = {"out": 0.0, "probs_abs": 0.0, "dq": 0.0, "dk": 0.0, "dv": 0.0}
    checked = 0
    for li in (0, len(layers) - 1):
        ly = layers[li]
        for item in sorted(set(rng.integers(0, B * Z, heads_per_layer).tolist()) | {B * Z - 1}):
            b, z = divmod(int(item), Z)
            f = lambda t: torch.cat([t[d, b, z] for d in range(t.shape[0])], 0).double().cpu().numpy()  # noqa: E731
            q, k, v, g = (f(ly[x]) for x in ("q", "k", "v", "g"))
            seq = q.shape[0]
            want = orc.attention_head_sampled(q, k, v, g, np.arange(seq), np.arange(seq))
            got = {"out": f(ly["o"]), "dq": f(ly["grads"][0]), "dk": f(ly["grads"][1]), "dv": f(ly["grads"][2])}
            for key, val in got.items():
                ref = want[key]
                worst[key] = max(worst[key], float(np.linalg.norm(val - ref) / np.linalg.norm(ref)))
            if "p" in ly:
                p = torch.cat([engine.normalized_panel(ly["p"][d, b, z], ly["r"][d, b, z]) for d in range(
                    ly["p"].shape[0])], 0).double().cpu().numpy()
            else:  # stream mode: the head's panel recomputed from its saved row statistics
                hd = lambda t: t[:, b:b + 1, z:z + 1]  # noqa: E731
                p = torch.cat([engine.stream_panel(hd(ly["q"]), hd(ly["k"]), hd(ly["v"]), hd(ly["m"]).contiguous(),
                                                   hd(ly["r"]).contiguous(), d)[0, 0] for d in range(ly["q"].shape[0])],
                              0).double().cpu().numpy()
            worst["probs_abs"] = max(worst["probs_abs"], float(np.max(np.abs(p - want["probs"]))))
            checked += 1
    ok = all(worst[k] <= 1e-2 for k in ("out", "dq", "dk", "dv")) and worst["probs_abs"] <= 4e-3
    return {"heads_checked": checked, "layers": [0, len(layers) - 1], "max_error": worst, "pass": ok,
            "gates": "out, dq, dk, dv: relative Frobenius error <= 1e-2; probs_abs: max |diff| of the "
                     "materialised probability rows <= 4e-3",
            "oracle": "oracle/ringseq_np.py attention_head_sampled (float64), same bf16 inputs"}


def e2e_public_api(args, dev):
    """Same step through ring_attention_forward/backward with pinned host buffers."""
    os.environ["RSA_B200_CHECK"] = args.e2e_checks
    try:
        return _e2e_public_api(args, dev)
    finally:
        os.environ.pop("RSA_B200_CHECK", None)


def _e2e_public_api(args, dev):
    import torch

    from paper_2105_13120_b200 import AttentionConfig
    from paper_2105_13120_b200.ring_attention import ring_attention_backward, ring_attention_forward

    B, Z, L, A, LAYERS = args.batch, args.heads, args.seq, args.head_size, args.layers
    R = args.ring_ranks
    c = L // R
    cfg = AttentionConfig(batch_size=B, seq_len=L, hidden_size=Z * A, num_heads=Z, head_size=A, num_devices=R)
    ch = lambda t: [t[:, :, d * c:(d + 1) * c] for d in range(R)]  # noqa: E731  (contiguous L/R chunks)
    cat_seq = lambda xs: xs[0] if R == 1 else torch.cat(xs, 2)  # noqa: E731
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
                fwd = ring_attention_forward(ch(q), ch(k), ch(v), cfg, mode=args.attn)
                outs[0].copy_(cat_seq(fwd.outputs), non_blocking=True)
            saved.append(fwd)
        if prefetch_next:
            upload(1 - set_i)
        for i in reversed(range(LAYERS)):
            q, k, v, gr = bufs[set_i][i]
            outs = host[i][1]
            st = streams[i % 2]
            with torch.cuda.stream(st):
                bwd = ring_attention_backward(ch(q), ch(k), ch(v), saved[i].probs, ch(gr), cfg)
                outs[1].copy_(cat_seq(bwd.grad_q), non_blocking=True)
                outs[2].copy_(cat_seq(bwd.grad_k), non_blocking=True)
                outs[3].copy_(cat_seq(bwd.grad_v), non_blocking=True)
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
                    "pinned host; layers alternate over 2 compute streams; status flags: " + args.e2e_checks}


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
    else:
        ours(args)


if __name__ == "__main__":
    main()
