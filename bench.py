"""bench.py — MCA attention-layer throughput on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c2|c1|c3|c4] [--alpha A] [--dtype bf16|f32]

One step = one MCA attention-layer forward over one batch of synthetic
BERT-shaped inputs already resident in HBM: the Q/K projections (q = x W_q,
k = x W_k: the reference's mca_forward(x, weights) takes x),
the score pass + Eq. 9 budgets, the sampled encoding and A.H~. Default
workload: BASELINE.json configs[1] — BERT-base (d=768, 12 heads of 64), B=64
sequences of n=512 per GPU, bf16, alpha=0.4. `--inputs qkx` gives q and k as
inputs instead (the default for the 24-layer c3 stack, whose layers chain
y -> x).

Multi-GPU (torchrun, one process per GPU): every rank runs its own B=64
sequences with b_offset = rank*B (weak scaling; no collective in the hot
path). Time = max over ranks of the device-timed total; NCCL is used only for
the barrier/max and, after timing, to gather per-rank checksums for
validation.

The JSON line also carries:
  e2e           the same metric through the C ABI with HOST buffers: pinned
                H2D of the step's inputs (x; q, k too with --inputs qkx), the
                forward, D2H of y inside the timed region, every step
                (HostPipeline: 4 batch chunks whose copies and forward overlap
                on three streams)
  roofline      the dominant kernel's achieved algorithmic GB/s or TFLOP/s vs
                MEASURED_PEAKS.json (DESIGN.md §7 defines the per-unit work)
  cpu_baseline  the fp64 CPU oracle (the reference algorithm, test
                infrastructure) on this host's cores, bounded sample
  clocks        nvidia-smi samples taken while the benchmark ran
`--impl reference` times the CPU reference path (the oracle port; the
reference itself ships no definitions) on the same config, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MCA attn-layer tokens/sec @BERT-base/large 1/2/4/8 B200; HBM GB/s frac; FLOP cut"

INPUTS_DESC = {
    "qkx": "q, k, x (the caller's Q/K projections given)",
    "x": "x only; q = x W_q, k = x W_k on the device (the reference's mca_forward(x, weights))",
}

CONFIGS = {
    # name: (B per GPU, n, d_in, heads, description)
    "c1": (1, 128, 768, 12, "BERT-base MCA attention layer, B=1, n=128 (configs[0])"),
    "c2": (64, 512, 768, 12, "BERT-base MCA attention layer, B=64, n=512, 1 B200 per 64 sequences (configs[1])"),
    "c3": (128, 512, 1024, 16, "BERT-large 24-layer MCA attention stack, B=128, n=512 (configs[2])"),
    "c4": (16, 4096, 768, 12, "long-sequence BERT-base MCA layer, B=16, n=4096 (configs[3])"),
}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return {"hbm_gbs": p["hbm_gbs"], "bf16_tflops": p["bf16_tflops"], "src": "measured"}
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "src": "fallback"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, device_index: int):
        self.idx = device_index
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        time.sleep(0.05)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        load = [v for v in sm if v > 0.5 * (max(sm) if sm else 1)]
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ----------------------------------------------------------------- CPU legs
def cpu_reference_rate(cfg_name: str, alpha: float, budget_s: float, threads: int, inputs: str = "qkx"):
    """Tokens/s of the fp64 CPU oracle (oracle/, the reference algorithm) on a
    bounded sample of the workload: whole sequences until ~budget_s seconds.
    inputs == "x": the projections q = x W_q, k = x W_k are part of the timed
    work (numpy fp64 matmul on all threads, a strong CPU GEMM)."""
    import numpy as np
    from oracle import oracle as orc
    from paper_2201_12854_b200 import synthetic
    B, n, d_in, H, _ = CONFIGS[cfg_name]
    orc.set_threads(threads)
    w = synthetic.make_weights(d_in, H).double().numpy()
    done_tokens, t_total, b = 0, 0.0, 0
    per = max(1, threads)  # sequences per call: keep every thread busy on (b, h) pairs
    while t_total < budget_s and b < 4 * B:
        if inputs == "x":
            pin = synthetic.make_projected_inputs(per, n, d_in, H, seed=1234 + b)
            x, wq, wk = (t.double().numpy() for t in (pin.x, pin.w_q, pin.w_k))
            t0 = time.perf_counter()
            q, k = np.matmul(x, wq), np.matmul(x, wk)
        else:
            inp = synthetic.make_inputs(per, n, d_in, H, seed=1234 + b)
            q, k, x = (t.double().numpy() for t in (inp.q, inp.k, inp.x))
            t0 = time.perf_counter()
        orc.batched_forward(q, k, x, w, heads=H, alpha=alpha, seed=42, b_offset=b, want_h=False)
        t_total += time.perf_counter() - t0
        done_tokens += per * n
        b += per
    proj = " incl. q = x W_q, k = x W_k (numpy)" if inputs == "x" else ""
    return (done_tokens / t_total, f"{b} sequences of n={n} ({done_tokens} tokens){proj}, fp64, {threads} threads",
            t_total)


def run_reference(args, rank: int):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    B, n, d_in, H, desc = CONFIGS[args.config]
    per_step_budget = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    rates = []
    for i in range(args.warmup + args.steps):
        r, sample, _ = cpu_reference_rate(args.config, args.alpha, per_step_budget, threads, args.inputs)
        if i >= args.warmup:
            rates.append(r)
    value = statistics.median(rates)
    line = {"metric": METRIC, "impl": "reference", "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * B * n / value,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "layers": args.layers, "global_batch": B * max(1, args.gpus), "B_per_gpu": B,
                       "seq_len": n, "d_in": d_in, "heads": H, "d_h": 64, "alpha": args.alpha, "seed": 42,
                       "parallelism": f"dp{max(1, args.gpus)} (batch shards)", "inputs": INPUTS_DESC[args.inputs],
                       "reference_sample": "bounded CPU sample per step, timed on this host's cores"},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "reference ships declarations only (matrix.hpp); the CPU reference path is the fp64 SPEC "
                    "restatement in oracle/ (OpenMP over (b, h)), timed on this host's cores"}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU leg
def algorithmic_work(B, n, d_in, H, elem, project: bool = False):
    dh = 64
    flops_qk = 2.0 * B * H * n * n * dh
    flops_proj = 2.0 * 2.0 * B * n * d_in * H * dh if project else 0.0   # q = x W_q, k = x W_k
    k3_bytes = B * n * d_in * elem + B * n * H * dh * elem + 4.0 * B * H * n + H * d_in * (dh * elem + 12)
    k2_bytes = B * H * n * (8 + 4 + 1)
    return {"score": ("tensor", flops_qk + flops_proj), "budgets": ("hbm", k2_bytes), "encode": ("hbm", k3_bytes),
            "apply": ("tensor", flops_qk)}


def run_ours(args, rank: int, world: int, local_rank: int):
    import torch

    import paper_2201_12854_b200 as mca
    from paper_2201_12854_b200.pipeline import HostPipeline
    from paper_2201_12854_b200 import synthetic

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    B, n, d_in, H, desc = CONFIGS[args.config]
    dtype = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    elem = 2 if dtype == torch.bfloat16 else 4
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    L = args.layers
    # per-layer W_V (seeded by layer); Q/K are the caller's projections (out of the
    # path): one synthetic set shared by the layers; layer l uses
    # Philox counter word `layer = l`, and X_{l+1} = Y_l chains the stack.
    wl = [synthetic.make_weights(d_in, H, seed=1234 + l).to(dtype) for l in range(L)]
    w = wl[0]
    project = args.inputs == "x"
    if project:   # x in, W_q / W_k with the weights: the reference's mca_forward(x, weights, ...)
        if L != 1:
            raise SystemExit("--inputs x runs one layer (the synthetic projections model layer-0 statistics)")
        pin = synthetic.make_projected_inputs(B, n, d_in, H, seed=1234 + rank)
        layer_weights = [mca.AttentionWeights(wl[0].to(dev), heads=H, w_q=pin.w_q.to(dtype).to(dev),
                                              w_k=pin.w_k.to(dtype).to(dev))]
        q = k = None
        x = pin.x.to(dtype).to(dev)
        host_inputs = (pin.x,)
    else:
        inp = synthetic.make_inputs(B, n, d_in, H, seed=1234 + rank)  # rank's own shard of the global batch
        layer_weights = [mca.AttentionWeights(t.to(dev), heads=H) for t in wl]
        q, k, x = (t.to(dtype).to(dev) for t in (inp.q, inp.k, inp.x))
        host_inputs = (inp.q, inp.k, inp.x)
    weights = layer_weights[0]
    y = torch.empty((B, n, H * 64), dtype=dtype, device=dev)
    ybuf = [torch.empty_like(y), torch.empty_like(y)]
    cfg = mca.McaConfig(alpha=args.alpha)
    b_offset = rank * B
    for lw in layer_weights:
        lw.reserve(B * n)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream()

    def step():
        # NVTX range "mca_step": the profiling scripts restrict ncu to the
        # device-resident steps (ncu --nvtx --nvtx-include "mca_step/"), so the
        # launch list is not mixed with the e2e leg's chunked launches
        torch.cuda.nvtx.range_push("mca_step")
        if L == 1:
            mca.mca_forward(weights, q, k, x, cfg, seed=42, b_offset=b_offset, y=y)
        else:
            xin = x
            for l in range(L):
                out_buf = ybuf[l & 1]
                mca.mca_forward(layer_weights[l], q, k, xin, cfg, seed=42, b_offset=b_offset, layer=l, y=out_buf)
                xin = out_buf
        torch.cuda.nvtx.range_pop()

    out = mca.mca_forward(weights, q, k, x, cfg, seed=42, b_offset=b_offset, y=y, flops=True, return_plan=True)
    flops_report = out.flops
    launches_per_step = weights.last_launch_count() * L

    sampler = ClockSampler(local_rank) if rank == 0 else None
    if sampler:
        sampler.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    # the timed steps carry no per-stage events (an event between two kernels
    # would stop the next one from starting early: programmatic dependent launch)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    for i in range(args.steps):
        flush.zero_()                                   # L2 flushed between timed steps (untimed)
        starts[i].record(stream)
        step()
        ends[i].record(stream)
    torch.cuda.synchronize()
    total_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    if dist:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    # per-stage device times (roofline / stages_ms): separate steps with the
    # forward's stage events on, same L2 flush
    for lw in layer_weights:
        lw.set_timing(True)
    stage_tot = [0.0, 0.0, 0.0, 0.0]
    for i in range(args.steps):
        flush.zero_()
        step()
        for lw in layer_weights:
            st = lw.last_stage_ms()                     # events on the forward's own stream
            for s in range(len(st)):
                stage_tot[s] += st[s]
    torch.cuda.synchronize()
    for lw in layer_weights:
        lw.set_timing(False)
    ms_per_step = total_ms / args.steps
    value = world * B * n * L / (ms_per_step / 1e3)   # token-layers per second (= tokens/s for one layer)

    # e2e: host buffers through the package's pipelined host API (HostPipeline:
    # every step copies its q, k, x from pinned host memory and reads y back,
    # in chunks whose H2D / forward / D2H overlap on three streams)
    if project:
        hq = hk = None
        hx = pin.x.to(dtype).pin_memory()
    else:
        hq, hk, hx = (t.to(dtype).pin_memory() for t in (inp.q, inp.k, inp.x))
    hy = torch.empty(y.shape, dtype=dtype).pin_memory()
    # chunking: a PCIe-bound step (device time under half the transfer time at ~50 GB/s)
    # overlaps best in 8 chunks with 4 in flight; a compute-bound one (C3's 24
    # layers, fp32, long sequences) in 4 chunks with 3 in flight (smaller chunks
    # cost kernel efficiency there). --e2e-chunks / --e2e-depth override.
    xfer_ms = (sum(t.numel() for t in host_inputs) + y.numel()) * elem / 50e9 * 1e3
    pcie_bound = ms_per_step < 0.5 * xfer_ms
    want = args.e2e_chunks or (8 if pcie_bound else 4)
    depth = args.e2e_depth or (4 if pcie_bound else 3)
    nch = want if B % want == 0 else 1
    chunk = B // nch
    pipe = HostPipeline(layer_weights, n, chunk, dtype, dev, depth=depth)

    def e2e_step():
        pipe.forward(hq, hk, hx, hy, cfg, seed=42, b_offset=b_offset)

    for _ in range(max(1, args.warmup)):
        e2e_step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    if dist:
        t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    clocks = sampler.stop() if sampler else None

    # validation gather (outside timing): per-rank checksums of y and the plan
    chk = torch.tensor([float(y.double().sum()), float(out.budgets.double().sum())], device=dev, dtype=torch.float64)
    if dist:
        allc = [torch.empty_like(chk) for _ in range(world)]
        dist.all_gather(allc, chk)
        checksums = [c.tolist() for c in allc]
    else:
        checksums = [chk.tolist()]

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    peaks = _peaks()
    work = {k: (v[0], v[1] * L) for k, v in algorithmic_work(B, n, d_in, H, elem, project).items()}   # per step
    names = ["score", "budgets", "encode", "apply"]
    stage_ms = {names[i]: stage_tot[i] / args.steps for i in range(4)}
    dom = max(names, key=lambda s: stage_ms[s])
    bound, amount = work[dom]
    if bound == "tensor":
        achieved = amount / (stage_ms[dom] / 1e3) / 1e12
        roof = {"kernel": dom, "bound": "tensor", "achieved": achieved, "peak": peaks["bf16_tflops"],
                "unit": "TFLOP/s", "frac": achieved / peaks["bf16_tflops"]}
    else:
        achieved = amount / (stage_ms[dom] / 1e3) / 1e9
        roof = {"kernel": dom, "bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"]}
    roof["peak_src"] = peaks["src"]
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(dom)
        except Exception:
            traffic = None
    roof["traffic"] = traffic
    enc_gbs = work["encode"][1] / (stage_ms["encode"] / 1e3) / 1e9
    gather_gbs = L * flops_report.samples * 64 * elem / (stage_ms["encode"] / 1e3) / 1e9   # layer 0's sample count x L

    cpu = None   # the CPU baseline runs on rank 0 at N = 1 only (multi-GPU lines carry null)
    if not args.no_cpu_baseline and world == 1:
        threads = os.cpu_count() or 1
        rate, sample, _ = cpu_reference_rate(args.config, args.alpha, args.cpu_seconds, threads, args.inputs)
        cpu = {"value": rate, "unit": "tokens/s (one layer)", "cores": threads, "kind": "port", "sample": sample}

    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        "config": {"workload": desc, "layers": L, "global_batch": world * B, "B_per_gpu": B, "seq_len": n, "d_in": d_in,
                   "heads": H, "d_h": 64, "alpha": args.alpha, "seed": 42, "parallelism": f"dp{world} (batch shards)",
                   "l2": "flushed (256 MB write) before every timed step", "inputs": INPUTS_DESC[args.inputs],
                   "e2e_pipeline": f"{nch} chunks, {depth} in flight"},
        "e2e": {"value": world * B * n * L / (e2e_ms / 1e3), "unit": "tokens/s",
                "h2d_bytes_per_step": int(sum(t.numel() for t in host_inputs) * elem),
                "d2h_bytes_per_step": int(y.numel() * elem)},
        "roofline": roof,
        "stages_ms": stage_ms,
        "encode": {"algorithmic_GBps": enc_gbs, "hbm_frac": enc_gbs / peaks["hbm_gbs"], "gather_GBps": gather_gbs,
                   "samples_per_step": flops_report.samples, "exact_token_heads": flops_report.exact_tokens},
        "flop_cut": {"reduction_factor": flops_report.reduction_factor,
                     "total_reduction": flops_report.total_reduction},
        "gpu_launches": launches_per_step * args.steps,
        "cpu_baseline": cpu,
        "clocks": clocks,
        "validation": {"rank_checksums": checksums},
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--alpha", type=float, default=0.4)
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "f32"])
    ap.add_argument("--layers", type=int, default=0, help="layers per step (default: 24 for c3, else 1)")
    ap.add_argument("--batch", type=int, default=0, help="override B per GPU")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-chunks", type=int, default=0, help="HostPipeline chunks per step (e2e leg; 0: auto)")
    ap.add_argument("--e2e-depth", type=int, default=0, help="HostPipeline device slots in flight (e2e leg; 0: auto)")
    ap.add_argument("--inputs", default=None, choices=sorted(INPUTS_DESC),
                    help="x: x alone, q/k projected on the device (default for one-layer configs: the "
                         "reference's mca_forward(x, weights)); qkx: q, k, x given (default for the c3 stack)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.layers <= 0:
        args.layers = 24 if args.config == "c3" else 1
    if args.inputs is None:
        args.inputs = "x" if args.layers == 1 else "qkx"
    if args.batch > 0:
        B, n, d_in, H, desc = CONFIGS[args.config]
        CONFIGS[args.config] = (args.batch, n, d_in, H, desc + f" [B overridden to {args.batch}]")
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
