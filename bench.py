"""bench.py — MCA attention-layer throughput on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c2|c1|c3|c4] [--alpha A] [--dtype bf16|f32]
                  [--global-batch G] [--layers L] [--inputs x|qkx]

One step = one MCA attention-layer forward (or, for c3, the 24-layer stack)
over one batch of synthetic BERT-shaped inputs already resident in HBM: the
Q/K projections (q = x W_q, k = x W_k on tcgen05: the reference's
mca_forward(x, weights) takes x), the score pass + Eq. 9
budgets (+ the binary64 certification of boundary cases), the sampled
encoding and A.H~. Default workload: BASELINE.json configs[1] — BERT-base
(d=768, 12 heads of 64), B=64 sequences of n=512 per GPU, bf16, alpha=0.4.
c1 runs in fp32 (configs[0] is fp32). c3 is the BERT-large stack: 24 layers,
each with its own W_q, W_k, W_V, chained X_{l+1} = Y_l, global batch 128
split over the ranks (strong scaling). `--inputs qkx` gives q and k as inputs
instead of x.

Multi-GPU: `--gpus N` without a torchrun environment re-launches itself under
torch.distributed.run with N ranks (one process per GPU); it refuses to run on
a box with fewer than N GPUs. Rank r runs its own batch shard with
b_offset = its first global sequence (no collective in the hot path). Time =
max over ranks of the device-timed total; NCCL is used only for the
barrier/max and, after timing, to gather per-rank checksums for validation.

The JSON line also carries:
  e2e           the same metric through the C ABI with HOST buffers: pinned
                H2D of the step's inputs, the forward, D2H of y inside the
                timed region, every step (HostPipeline: batch chunks whose
                copies and forward overlap on three streams)
  roofline      the dominant stage's achieved algorithmic GB/s or TFLOP/s vs
                MEASURED_PEAKS.json (DESIGN.md §7 defines the per-unit work)
  kernels       every stage against its roofline and the floors that bind it
                (MUFU exponentials, shared-memory wavefronts, FMA issue)
  regular       the exact layer (regular_forward) on the same inputs: its time
                and the MCA layer's wall-clock speed-up over it
  cpu_baseline  the fp64 CPU oracle (the reference algorithm, test
                infrastructure) on this host's cores, bounded sample; the same
                leg checks the device budgets against the oracle's on the
                device's own inputs (budget_mismatch_vs_fp64)
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
    "c1": (1, 128, 768, 12, "BERT-base MCA attention layer, B=1, n=128, fp32 (configs[0])"),
    "c2": (64, 512, 768, 12, "BERT-base MCA attention layer, B=64, n=512, 1 B200 per 64 sequences (configs[1])"),
    "c3": (128, 512, 1024, 16, "BERT-large 24-layer MCA attention stack, global B=128, n=512, batch-sharded (configs[2])"),
    "c4": (16, 4096, 768, 12, "long-sequence BERT-base MCA layer, B=16, n=4096 (configs[3])"),
}
DEFAULT_DTYPE = {"c1": "f32"}          # BASELINE.json configs[0] is fp32; the others bf16
DEFAULT_GLOBAL_BATCH = {"c3": 128}     # c3: batch 128 sharded across the GPUs (strong scaling)


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


def _shard(args, rank: int, world: int):
    """(B on this rank, b_offset, global batch, scaling) for the config:
    weak scaling keeps B per GPU fixed; --global-batch splits a fixed batch."""
    from paper_2201_12854_b200 import sharding
    B, n, d_in, H, desc = CONFIGS[args.config]
    if args.global_batch > 0:
        start, count = sharding.shard_range(args.global_batch, rank, world)
        return count, start, args.global_batch, "strong"
    return B, rank * B, B * world, "weak"


def _config_dict(args, world, B, GB):
    _, n, d_in, H, desc = CONFIGS[args.config]
    return {"workload": desc, "layers": args.layers, "global_batch": GB, "B_per_gpu": B, "seq_len": n,
            "d_in": d_in, "heads": H, "d_h": 64, "alpha": args.alpha, "seed": 42, "certify": bool(args.certify),
            "parallelism": f"dp{world} (batch shards)", "inputs": INPUTS_DESC[args.inputs]}


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    B, n, d_in, H, desc = CONFIGS[args.config]
    nw = max(world, args.gpus)
    Bq, _, GB, scaling = _shard(args, 0, nw)
    per_step_budget = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    rates = []
    for i in range(args.warmup + args.steps):
        r, sample, _ = cpu_reference_rate(args.config, args.alpha, per_step_budget, threads, args.inputs)
        if i >= args.warmup:
            rates.append(r)
    value = statistics.median(rates)   # tokens/s per layer = token-layers/s of an L-layer stack
    cfg = _config_dict(args, nw, Bq, GB)
    cfg["reference_sample"] = "bounded CPU sample per step, timed on this host's cores"
    line = {"metric": METRIC, "impl": "reference", "value": value, "unit": "tokens/s", "n_gpus": nw,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * GB * n * args.layers / value,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": cfg,
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "reference ships declarations only (matrix.hpp); the CPU reference path is the fp64 SPEC "
                    "restatement in oracle/ (OpenMP over (b, h)), timed on this host's cores"}
    print(json.dumps(line), flush=True)


def budget_parity_sample(mca, weights, x, q, k, cfg, n, d_in, H, b_offset, seqs: int, threads: int):
    """The cpu_baseline leg's check of the timed workload: one more forward
    (untimed) returns the device's plan and, for x inputs, its projected q, k;
    the fp64 oracle runs on the first `seqs` sequences of those same (bf16 /
    fp32) inputs and its end-to-end budgets are compared with the device's
    (SURVEY.md §8(c)(5)): count, and distance of the oracle's raw value to the
    integer boundary for any mismatch."""
    import numpy as np
    import torch
    from oracle import oracle as orc
    S = min(seqs, x.shape[0])
    xs = x[:S].contiguous()
    dbg = {}
    if q is None:
        dbg = dict(q_out=torch.empty((S, n, H * 64), dtype=x.dtype, device=x.device),
                   k_out=torch.empty((S, n, H * 64), dtype=x.dtype, device=x.device))
        out = mca.mca_forward(weights, None, None, xs, cfg, seed=42, b_offset=b_offset, return_plan=True, debug=dbg)
        qs, ks = dbg["q_out"], dbg["k_out"]
    else:
        qs, ks = q[:S].contiguous(), k[:S].contiguous()
        out = mca.mca_forward(weights, qs, ks, xs, cfg, seed=42, b_offset=b_offset, return_plan=True)
    torch.cuda.synchronize()
    f64 = lambda t: t.detach().double().cpu().numpy()   # noqa: E731
    orc.set_threads(threads)
    ref = orc.batched_forward(f64(qs), f64(ks), f64(xs), f64(weights_w(weights)), heads=H, alpha=cfg.alpha, seed=42,
                              b_offset=b_offset, want_h=False)
    b = out.budgets.cpu().numpy()
    e = out.exact_mask.cpu().numpy().astype(bool)
    mism = (b != ref.budgets) | (e != ref.exact)
    dist = 0.0
    if mism.any():
        t = (float(n) * ref.cmax[mism]) / cfg.alpha
        bound = np.minimum(b[mism], ref.budgets[mism]).astype(np.float64)
        dist = float((np.abs(t * t - bound) / np.maximum(bound, 1.0)).max())
    return {"count": int(mism.sum()), "checked_token_heads": int(b.size), "max_dist_to_int": dist,
            "sample": f"first {S} sequences of the timed batch, layer 0, device q/k/x vs the fp64 oracle"}


def weights_w(weights):
    return weights._bench_w


# ---------------------------------------------------------------- GPU leg
def stage_work(B, n, d_in, H, elem, project: bool, samples: int):
    """Algorithmic work per stage of one layer: flops for
    tensor-core stages, bytes for HBM stages, and the floors that bind the
    non-GEMM work (MUFU exponentials, shared-memory wavefronts, FMA issue)."""
    dh = 64
    flops_qk = 2.0 * B * H * n * n * dh
    return {
        "projection": ("tensor", 2.0 * 2.0 * B * n * d_in * H * dh if project else 0.0),
        "score": ("tensor", flops_qk),
        "budgets": ("hbm", B * H * n * (8 + 4 + 1)),
        "encode": ("hbm", B * n * d_in * elem + B * n * H * dh * elem + 4.0 * B * H * n + H * d_in * (dh * elem + 12)),
        "apply": ("tensor", flops_qk),
        "_exps": float(B * H * n * n),          # one exponential per score (score pass; K4 again)
        "_samples": float(samples),
    }


def kernel_table(work, stage_ms, peaks, clk_mhz, sms=148):
    """Per stage: achieved vs its roofline, and the fraction of the floor that
    binds it in practice."""
    clk = (clk_mhz or 1965.0) * 1e6
    out = {}
    for name, spec in work.items():
        if name.startswith("_"):
            continue
        bound, amount = spec
        if name not in stage_ms or stage_ms[name] <= 0 or amount <= 0:
            continue
        t = stage_ms[name] / 1e3
        if bound == "tensor":
            ach = amount / t / 1e12
            e = {"ms": stage_ms[name], "bound": "tensor", "achieved": ach, "unit": "TFLOP/s",
                 "peak": peaks["bf16_tflops"], "frac": ach / peaks["bf16_tflops"]}
        else:
            ach = amount / t / 1e9
            e = {"ms": stage_ms[name], "bound": "hbm", "achieved": ach, "unit": "GB/s", "peak": peaks["hbm_gbs"],
                 "frac": ach / peaks["hbm_gbs"]}
        if name == "score":      # row statistics: one ex2 per score on the MUFU (16 / clk / SM)
            fl = work["_exps"] / (sms * 16 * clk)
            e["mufu_floor_ms"] = fl * 1e3
            e["frac_of_mufu_floor"] = fl / t
        if name == "apply":      # P = 2^(cS - lse): ex2.approx.f16x2, two exponentials per MUFU op
            fl = work["_exps"] / 2 / (sms * 16 * clk)
            e["mufu_floor_ms"] = fl * 1e3
            e["frac_of_mufu_floor"] = fl / t
        if name == "encode" and work["_samples"] > 0:   # 128-byte W row read + 64 MACs per sample
            smem = work["_samples"] / (sms * clk)              # one 128 B wavefront per sample, 1 / clk / SM
            fma = work["_samples"] * 64 / (sms * 128 * clk)    # 128 FMA lanes / clk / SM
            e.update({"smem_floor_ms": smem * 1e3, "frac_of_smem_floor": smem / t, "fma_floor_ms": fma * 1e3,
                      "frac_of_fma_floor": fma / t})
        out[name] = e
    return out


def run_ours(args, rank: int, world: int, local_rank: int):
    import torch

    import paper_2201_12854_b200 as mca
    from paper_2201_12854_b200.pipeline import HostPipeline
    from paper_2201_12854_b200 import synthetic

    # MCA_BENCH_SHARED_GPU=1 (functional tests of the N > 1 plumbing on a 1-GPU
    # box only: every rank on device 0 over gloo; never a reported number)
    shared = os.environ.get("MCA_BENCH_SHARED_GPU") == "1"
    if torch.cuda.device_count() <= local_rank and not shared:
        raise SystemExit(f"rank {rank}: local rank {local_rank} but only {torch.cuda.device_count()} CUDA device(s)")
    dev_index = 0 if shared else local_rank
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    _, n, d_in, H, desc = CONFIGS[args.config]
    B, b_offset, GB, scaling = _shard(args, rank, world)
    dtype = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    elem = 2 if dtype == torch.bfloat16 else 4
    dist = None
    if world > 1:
        import torch.distributed as dist
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    L = args.layers
    project = args.inputs == "x"
    # layer l: its own W_V (seed 1234 + l) and, for x inputs, its own W_q / W_k
    # (the sink-model projections of synthetic.make_projected_inputs); layer l
    # uses Philox counter word `layer = l`, and X_{l+1} = Y_l chains the stack
    wl = [synthetic.make_weights(d_in, H, seed=1234 + l).to(dtype) for l in range(L)]
    if project:
        if scaling == "strong":   # every rank slices the same global batch
            pin = synthetic.make_projected_inputs(GB, n, d_in, H, seed=1234)
            x_host = pin.x[b_offset:b_offset + B].contiguous()
        else:
            pin = synthetic.make_projected_inputs(B, n, d_in, H, seed=1234 + rank)
            x_host = pin.x
        layer_weights = []
        for l in range(L):
            pl = pin if l == 0 else synthetic.make_projected_inputs(1, 1, d_in, H, seed=1234 + l)
            layer_weights.append(mca.AttentionWeights(wl[l].to(dev), heads=H, w_q=pl.w_q.to(dtype).to(dev),
                                                      w_k=pl.w_k.to(dtype).to(dev)))
        q = k = None
        x = x_host.to(dtype).to(dev)
        host_inputs = (x_host,)
    else:
        if scaling == "strong":
            inp = synthetic.make_inputs(GB, n, d_in, H, seed=1234)
            sl = slice(b_offset, b_offset + B)
            inp = synthetic.LayerInputs(inp.q[sl].contiguous(), inp.k[sl].contiguous(), inp.x[sl].contiguous())
        else:
            inp = synthetic.make_inputs(B, n, d_in, H, seed=1234 + rank)  # rank's own shard of the global batch
        layer_weights = [mca.AttentionWeights(t.to(dev), heads=H) for t in wl]
        q, k, x = (t.to(dtype).to(dev) for t in (inp.q, inp.k, inp.x))
        host_inputs = (inp.q, inp.k, inp.x)
    weights = layer_weights[0]
    weights._bench_w = wl[0]
    y = torch.empty((B, n, H * 64), dtype=dtype, device=dev)
    ybuf = [torch.empty_like(y), torch.empty_like(y)]
    cfg = mca.McaConfig(alpha=args.alpha, certify=args.certify)
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

    sampler = ClockSampler(dev_index) if rank == 0 else None
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
    # per-stage device times (roofline / kernels): separate steps with the
    # forward's stage events on, same L2 flush
    names = ["projection", "score", "budgets", "encode", "apply"]
    for lw in layer_weights:
        lw.set_timing(True)
    stage_tot = [0.0] * len(names)
    for i in range(args.steps):
        flush.zero_()
        step()
        for lw in layer_weights:
            st = lw.last_stage_ms()                     # events on the forward's own stream
            for s_ in range(min(len(st), len(names))):
                stage_tot[s_] += st[s_]
    torch.cuda.synchronize()
    for lw in layer_weights:
        lw.set_timing(False)
    ms_per_step = total_ms / args.steps
    value = GB * n * L / (ms_per_step / 1e3)   # token-layers per second (= tokens/s for one layer)

    # the exact layer on the same inputs (regular_forward):
    # what the MCA layer's FLOP cut is measured against, timed the same way
    regular = None
    if not args.no_regular:
        yr = torch.empty_like(y)
        for _ in range(2):
            mca.regular_forward(weights, q, k, x, y=yr)
        torch.cuda.synchronize()
        r0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        r1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        for i in range(args.steps):
            flush.zero_()
            r0[i].record(stream)
            mca.regular_forward(weights, q, k, x, y=yr)
            r1[i].record(stream)
        torch.cuda.synchronize()
        reg_ms = sum(a_.elapsed_time(b_) for a_, b_ in zip(r0, r1)) / args.steps
        regular = {"ms_per_layer": reg_ms, "mca_ms_per_layer": ms_per_step / L,
                   "mca_speedup": reg_ms / (ms_per_step / L)}

    # e2e: host buffers through the package's pipelined host API (HostPipeline:
    # every step copies its inputs from pinned host memory and reads y back,
    # in chunks whose H2D / forward / D2H overlap on three streams)
    if project:
        hq = hk = None
        hx = x_host.to(dtype).pin_memory()
    else:
        hq, hk, hx = (t.to(dtype).pin_memory() for t in host_inputs)
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
        # serving-style: back-to-back steps pipeline across steps (the next step's
        # H2D and forward overlap this step's D2H); every step still moves its
        # own x in and y out, and the timed region ends when the last y landed
        pipe.forward(hq, hk, hx, hy, cfg, seed=42, b_offset=b_offset, sync=False)

    for _ in range(max(1, args.warmup)):
        e2e_step()
    pipe.wait()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    pipe.wait()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    if dist:
        t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    clocks = sampler.stop() if sampler else None

    # validation (outside timing; NCCL only here): per-rank checksums of y and
    # the plan, and for one-layer configs the outputs themselves: rank 0 gathers
    # every shard's y and re-runs the LAST rank's shard on its own GPU from that
    # rank's seeded inputs and weights with the same b_offset -- the shard must
    # come back bitwise (Philox streams use the global sequence index)
    chk = torch.tensor([float(y.double().sum()), float(out.budgets.double().sum())], device=dev, dtype=torch.float64)
    validation = {}
    if dist:
        allc = [torch.empty_like(chk) for _ in range(world)]
        dist.all_gather(allc, chk)
        checksums = [c.tolist() for c in allc]
        if L == 1:
            from paper_2201_12854_b200 import sharding
            yall = sharding.gather_shards(y, GB, rank, world) if scaling == "strong" else None
            if scaling == "weak":
                bufs = [torch.empty_like(y) for _ in range(world)]
                dist.all_gather(bufs, y)
                yall = torch.cat(bufs)
            if rank == 0:
                r_last = world - 1
                s_last, c_last = _shard(args, r_last, world)[1], _shard(args, r_last, world)[0]
                if project:
                    pl = (synthetic.make_projected_inputs(B, n, d_in, H, seed=1234 + r_last) if scaling == "weak"
                          else pin)
                    xl = (pl.x if scaling == "weak" else pin.x[s_last:s_last + c_last]).to(dtype).to(dev)
                    wr = mca.AttentionWeights(wl[0].to(dev), heads=H, w_q=pl.w_q.to(dtype).to(dev),
                                              w_k=pl.w_k.to(dtype).to(dev))
                    yr = mca.mca_forward(wr, None, None, xl.contiguous(), cfg, seed=42, b_offset=s_last).y
                else:
                    il = (synthetic.make_inputs(B, n, d_in, H, seed=1234 + r_last) if scaling == "weak"
                          else synthetic.make_inputs(GB, n, d_in, H, seed=1234))
                    sl_ = slice(0, c_last) if scaling == "weak" else slice(s_last, s_last + c_last)
                    ql, kl, xl = (t[sl_].contiguous().to(dtype).to(dev) for t in (il.q, il.k, il.x))
                    yr = mca.mca_forward(weights, ql, kl, xl, cfg, seed=42, b_offset=s_last).y
                off = s_last if scaling == "strong" else r_last * B
                validation = {"gathered_y_bytes": int(yall.numel() * yall.element_size()),
                              "last_shard_recomputed_on_rank0_bitwise": bool(torch.equal(yr, yall[off:off + c_last]))}
    else:
        checksums = [chk.tolist()]

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    peaks = _peaks()
    work1 = stage_work(B, n, d_in, H, elem, project, flops_report.samples)
    stage_ms = {names[i]: stage_tot[i] / args.steps for i in range(len(names))}
    per_layer_ms = {k_: v / L for k_, v in stage_ms.items()}      # stage tables are per layer
    kernels = kernel_table(work1, per_layer_ms, peaks, (clocks or {}).get("sm_mhz"))
    dom = max((s_ for s_ in names if s_ in kernels), key=lambda s_: stage_ms[s_])
    roof = {k_: kernels[dom][k_] for k_ in ("bound", "achieved", "peak", "unit", "frac")}
    roof["kernel"] = dom
    roof["peak_src"] = peaks["src"]
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(dom)
        except Exception:
            traffic = None
    roof["traffic"] = traffic
    enc_t = per_layer_ms["encode"] / 1e3
    gather_gbs = flops_report.samples * 64 * elem / enc_t / 1e9 if enc_t > 0 else None

    cpu = None   # the CPU baseline runs on rank 0 at N = 1 only (multi-GPU lines carry null)
    parity = None
    if not args.no_cpu_baseline and world == 1:
        threads = os.cpu_count() or 1
        rate, sample, _ = cpu_reference_rate(args.config, args.alpha, args.cpu_seconds, threads, args.inputs)
        cpu = {"value": rate, "unit": "tokens/s (one layer)", "cores": threads, "kind": "port", "sample": sample}
        parity = budget_parity_sample(mca, weights, x, q, k, cfg, n, d_in, H, b_offset,
                                      args.parity_seqs, threads)

    cfgd = _config_dict(args, world, B, GB)
    cfgd.update({"l2": "flushed (256 MB write) before every timed step", "e2e_pipeline": f"{nch} chunks, {depth} in flight"})
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        "config": cfgd,
        "e2e": {"value": GB * n * L / (e2e_ms / 1e3), "unit": "tokens/s",
                "h2d_bytes_per_step": int(sum(t.numel() for t in host_inputs) * elem),
                "d2h_bytes_per_step": int(y.numel() * elem)},
        "roofline": roof,
        "kernels": kernels,
        "stages_ms": stage_ms,
        "encode": {"algorithmic_GBps": kernels.get("encode", {}).get("achieved"),
                   "hbm_frac": kernels.get("encode", {}).get("frac"), "gather_GBps": gather_gbs,
                   "samples_per_layer": flops_report.samples, "exact_token_heads": flops_report.exact_tokens},
        "flop_cut": {"reduction_factor": flops_report.reduction_factor,
                     "total_reduction": flops_report.total_reduction},
        "budget_certification": {"enabled": bool(args.certify),
                                 "token_heads_rederived_fp64": flops_report.certified,
                                 "token_heads": B * H * n, "layer": 0},
        "budget_mismatch_vs_fp64": parity,
        "regular": regular,
        "gpu_launches": launches_per_step * args.steps,
        "cpu_baseline": cpu,
        "clocks": clocks,
        "validation": {"rank_checksums": checksums, **validation},
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def _free_port() -> int:
    import socket
    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    p = s_.getsockname()[1]
    s_.close()
    return p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--alpha", type=float, default=0.4)
    ap.add_argument("--dtype", default=None, choices=["bf16", "f32"], help="default: f32 for c1, else bf16")
    ap.add_argument("--layers", type=int, default=0, help="layers per step (default: 24 for c3, else 1)")
    ap.add_argument("--batch", type=int, default=0, help="override B per GPU (weak scaling)")
    ap.add_argument("--global-batch", type=int, default=-1,
                    help="global batch split over the GPUs (strong scaling; default 128 for c3, else off)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--parity-seqs", type=int, default=4, help="sequences the budget parity check runs on")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-regular", action="store_true", help="skip timing the exact layer")
    ap.add_argument("--certify", action="store_true",
                    help="McaConfig(certify=True): boundary Eq. 9 values re-derived in binary64")
    ap.add_argument("--e2e-chunks", type=int, default=0, help="HostPipeline chunks per step (e2e leg; 0: auto)")
    ap.add_argument("--e2e-depth", type=int, default=0, help="HostPipeline device slots in flight (e2e leg; 0: auto)")
    ap.add_argument("--inputs", default="x", choices=sorted(INPUTS_DESC),
                    help="x: x alone, q/k projected on the device per layer (the reference's mca_forward(x, "
                         "weights)); qkx: q, k, x given")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.dtype is None:
        args.dtype = DEFAULT_DTYPE.get(args.config, "bf16")
    if args.layers <= 0:
        args.layers = 24 if args.config == "c3" else 1
    if args.global_batch < 0:
        args.global_batch = DEFAULT_GLOBAL_BATCH.get(args.config, 0) if args.batch <= 0 else 0
    if args.batch > 0:
        B, n, d_in, H, desc = CONFIGS[args.config]
        CONFIGS[args.config] = (args.batch, n, d_in, H, desc + f" [B per GPU overridden to {args.batch}]")
    under_launcher = "WORLD_SIZE" in os.environ
    if args.impl == "ours" and args.gpus > 1 and not under_launcher:
        # one process per GPU: re-launch under torch.distributed.run
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            raise SystemExit(f"bench.py --gpus {args.gpus}: this box has {have} CUDA device(s); refusing to "
                             f"report a {args.gpus}-GPU number measured on fewer GPUs")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "ours" and under_launcher and world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
