#!/usr/bin/env python
"""bench.py -- FloE compressed-expert decode on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--layers L] [--no-offload] [--no-cpu-baseline]

Workload (BASELINE.json configs[2], the largest single-GPU configuration):
full 32-layer Mixtral-8x7B-shaped decode -- every layer a MoE block (mixing
matrix stand-in for attention, router top-2 of 8 compressed experts: INT2 g64
up projection, f16 gate|down records, ~80% contextual sparsity), all 256
experts resident in HBM (65.9 GB).  A step is one decode token through the 32
layers (the reference's run loop, cli.cpp:86-107); value = decode tokens/s
over all ranks.  N > 1 runs N independent replicas ("replicas only":
single-sequence decode does not shard).

Block inputs (replay): layer l of token i reads its own recorded N(0,1) block
input token_input(1, 32 i + l).  The synthetic stack has no norms and its
chained activations overflow by layer ~7, so a decode whose
hidden states keep their scale is replayed layer by layer
(predictor.cpp:60-85); every launch still waits for the previous layer (stream
order + PDL), exactly as in a chained decode.  Thresholds: the reference's
calibrate_model(k = 0.8) per layer (64 calibration tokens token_input(3, t)
as block inputs), computed ON THE DEVICE by floe_gpu_calib_* (bit-exact with
the reference, tests/test_gpu_calib.py).

Sub-results: "layer" (config 2: the same launches per layer), "expert_ffn"
(config 1 and the config-4 batched expert), "offload" (config 3 with the
records host-resident under a VRAM budget: PCIe-bound), "e2e" (the decode
through the host-buffer C ABI).

Weights are the reference's own gen_model random streams (seed 7), generated
and quantized on the device by the product library.  L2: one token touches
5.27 GB of weights (> 126 MB L2), no flush needed.

Only the cpu_baseline leg and --impl reference touch oracle/ (the reference
core compiled from its own sources, oracle/_ref/libfloe_ref.so).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "decode tokens/s (Mixtral-8x7B shape) + expert-FFN achieved HBM GB/s vs roofline"
DH, DI, E, TOPK, BITS, G, KSP, SEED = 4096, 14336, 8, 2, 2, 64, 0.8, 7
N_CAL = 64                           # calibration tokens per layer
N_MODEL_LAYERS = 32
WORKLOAD = ("config3: 32-layer Mixtral-8x7B-shaped decode (d=4096, ffn=14336, 8 experts, top-2 "
            "per layer), INT2 g64 up + ~80% contextual gate/down sparsity, all 256 experts "
            "HBM-resident, batch 1")
REC_BYTES = 4 * DH                   # one f16 gate|down channel record
CODE_BYTES = DH * DI * BITS // 8     # 14,680,064
META_BYTES = 4 * (DH * DI // G)      # 3,670,016
MIX_BYTES = DH * DH * 2              # f16 mixing


def weight_stream(layer, kind, expert):  # core/src/model.cpp:25-28
    return ((layer * 5 + kind) * 65536 + expert) * 64


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                stderr=subprocess.DEVNULL)
            time.sleep(0.25)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.f.close()

    def summary(self) -> dict:
        if not self.path or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9 and parts[1].replace(".", "").isdigit():
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(float(r[1]) for r in rows),
                "sm_max_mhz": max(float(r[2]) for r in rows), "reasons": reasons,
                "samples": len(rows), "power_w_max": max(float(r[3]) for r in rows)}


# ------------------------------------------------------------------ distributed
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def max_over_ranks(value: float, world: int, device=None) -> float:
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def whole_job_value(world: int, units_per_rank: int, max_ms: float) -> float:
    """Whole-job throughput: the units ALL ranks processed over the slowest rank's time."""
    return world * units_per_rank / (max_ms / 1000.0)


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ------------------------------------------------------------------ our arm
def gen_float_layer(fb, layer_idx):
    """gen_model streams (model.cpp:25-74) of one layer as f32 device tensors."""
    sigma = float(np.float32(1.0) / np.sqrt(np.float32(DH)))
    g = lambda kind, e, n: fb.gen_normals(SEED, weight_stream(layer_idx, kind, e), n, sigma,  # noqa: E731
                                          sharded=True)
    router = g(0, 0, E * DH).view(E, DH)
    mixing = g(1, 0, DH * DH).view(DH, DH)
    gate = [g(2, e, DH * DI).view(DI, DH) for e in range(E)]
    up = [g(3, e, DH * DI).view(DI, DH) for e in range(E)]
    down = [g(4, e, DH * DI).view(DI, DH) for e in range(E)]
    return router, mixing, gate, up, down


def build_layer(fb, torch, layer_idx=0):
    """One compressed layer (thresholds 0; set by calibrate() / calibrate_layer())."""
    router, mixing, gate, up, down = gen_float_layer(fb, layer_idx)
    experts = []
    for e in range(E):
        codes, scales, zeros = fb.quantize(up[e].reshape(-1), BITS, G)
        experts.append(fb.GpuExpert(DH, DI, BITS, G, codes, scales, zeros, gate=gate[e],
                                    down=down[e], threshold=0.0))
    del gate, up, down
    torch.cuda.synchronize()
    return router, mixing, experts


def calibrate_layer(fb, torch, router, mixing, gate, up, down):
    """calibrate_model(k=0.8) of one layer as a 1-layer model, on the device
    (floe_gpu_calib_*; model.cpp:242-330): N_CAL block inputs token_input(3, t)."""
    cal = fb.GpuCalib(1, E, DH, DI, 3)
    h = torch.stack([fb.gen_normals(3, (1 << 40) + t, DH) for t in range(N_CAL)])
    cal.layer(0, router, mixing, gate, up, down, TOPK, h, want_next=False)
    th = cal.thresholds(KSP)[0]
    cal.close()
    return [float(t) for t in th]


def quantile_threshold(torch, mags, k):
    """calibrate_threshold (sparsify.cpp:42-54): sorted[ceil(k N) - 1]."""
    s, _ = torch.sort(mags)
    n = s.numel()
    rank = min(max(int(math.ceil(k * n)), 1), n)
    return float(s[rank - 1].item())


def calibrate(fb, torch, router, mixing, experts, ws, n_cal=8):
    """Quick per-expert thresholds for tools: 0.8-quantile of |qgemv(up_e, u)| over
    n_cal calibration tokens (the compressed up projection)."""
    mags = [[] for _ in experts]
    for t in range(n_cal):
        h = fb.gen_normals(3, (1 << 40) + t, DH)
        u = h + mixing @ h
        for e, ex in enumerate(experts):
            mags[e].append(fb.qgemv_channels(ex, u.contiguous(), ws).abs())
    ths = []
    for e, ex in enumerate(experts):
        th = quantile_threshold(torch, torch.cat(mags[e]), KSP)
        ex.set_threshold(th)
        ths.append(th)
    return ths


N_LAYERS = 4   # (tools) distinct layers cycled
N_EXPERTS_C1 = 4  # distinct config-1 experts cycled


def build_model(fb, torch, n_layers):
    """n_layers compressed layers of the seed-7 model, each calibrated on the device;
    returns GpuLayers, thresholds [L][E]."""
    layers, ths = [], []
    for li in range(n_layers):
        router, mixing, gate, up, down = gen_float_layer(fb, li)
        th = calibrate_layer(fb, torch, router, mixing, gate, up, down)
        experts = []
        for e in range(E):
            codes, scales, zeros = fb.quantize(up[e].reshape(-1), BITS, G)
            experts.append(fb.GpuExpert(DH, DI, BITS, G, codes, scales, zeros, gate=gate[e],
                                        down=down[e], threshold=th[e]))
        del gate, up, down
        layers.append(fb.GpuLayer(router, mixing, experts, TOPK, mixing_f16=True))
        del router, mixing
        ths.append(th)
    torch.cuda.synchronize()
    return layers, ths


def time_region(torch, fn, n, stream):
    """n back-to-back steps in ONE CUDA-event region on `stream` (ms)."""
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for i in range(n):
        fn(i)
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b)


def replay_inputs(fb, torch, n_tokens, n_layers, first=0):
    """[n_tokens][L][dh] block inputs token_input(1, L*i + l)."""
    return torch.stack([torch.stack([fb.gen_normals(1, (1 << 40) + n_layers * i + l, DH)
                                     for l in range(n_layers)])
                        for i in range(first, first + n_tokens)])


def run_offload(fb, torch, layers, ws, n_tokens, budget_gb, stream):
    """Config 3 host-resident: records in pinned host memory read in place over PCIe,
    whole experts promoted into an HBM cache under the VRAM budget."""
    L = len(layers)
    off = fb.Offload(layers, int(budget_gb * (1 << 30)))
    n_warm, n_eval = 10, 2
    hs = replay_inputs(fb, torch, n_warm + n_tokens + n_eval, L, first=1000)
    y = torch.empty(L, DH, device="cuda")
    for i in range(n_warm):  # the HBM cache fills (promotions) before the timed tokens
        off.decode_replay(hs[i], ws, out=y)
    torch.cuda.synchronize()
    s0 = off.stats()
    ms = time_region(torch, lambda i: off.decode_replay(hs[n_warm + i], ws, out=y), n_tokens,
                     stream)
    s1 = off.stats()
    # predictor scores on the decode path (untimed): reuse masks of layer l
    # from layer l-1's block input
    off.set_eval(True)
    for i in range(n_eval):
        off.decode_replay(hs[n_warm + n_tokens + i], ws, out=y)
    s2 = off.stats()
    off.close()
    rb = s1["record_bytes"]
    pcie = (s1["records_over_pcie"] - s0["records_over_pcie"]) * rb / n_tokens
    hbm_rec = (s1["records_from_hbm"] - s0["records_from_hbm"]) * rb / n_tokens
    sec = ms * 1e-3 / n_tokens
    tl = {k: s2[k] for k in ("bytes_demanded", "bytes_from_cache", "bytes_prefetch_used",
                             "bytes_sync", "bytes_prefetch_wasted", "bytes_prefetch_pending")}
    return {"workload": f"config3: {L}-layer decode, gate|down records host-resident "
                        f"(pinned, read in place over PCIe), HBM expert cache {budget_gb} GB",
            "tokens": n_tokens, "value": round(1.0 / sec, 3), "unit": "tokens/s",
            "ms_per_token": round(sec * 1e3, 3),
            "record_bytes_per_token_over_pcie": int(pcie),
            "record_bytes_per_token_from_hbm": int(hbm_rec),
            "pcie_gbs": round(pcie / sec / 1e9, 2),
            "promotions": s1["promotions"] - s0["promotions"],
            "warmup_tokens": n_warm,
            "timeline_all_tokens": tl,
            "reuse_mask_predictor": {
                "precision": round(s2["mask_precision"], 4), "recall": round(s2["mask_recall"], 4),
                "samples": s2["mask_samples"],
                "note": "replayed block inputs are independent N(0,1) draws per layer, so the "
                        "previous layer's input carries no information: chance level"}}


def run_ours(args, rank, world, local):
    import torch
    import torch.distributed as dist

    import paper_2505_05950_b200 as fb

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = fb.device_info()
    hbm_peak, peak_kind = peaks()
    stream = torch.cuda.current_stream()
    L = args.layers

    # ---------------- setup (untimed) ----------------
    t_setup = time.perf_counter()
    ws = fb.Workspace(DH, DI, TOPK)
    layers, thresholds = build_model(fb, torch, L)
    model = fb.GpuModel(layers)
    n_tok = args.warmup + args.steps
    hs = replay_inputs(fb, torch, n_tok, L)   # [tokens][L][dh]
    y = torch.empty(L, DH, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup

    def step(i, off=args.warmup):
        model.decode(hs[off + i], ws, out=y, replay=True)

    # ---------------- warmup + timed region ----------------
    time_region(torch, lambda i: step(i, 0), args.warmup, stream)
    barrier(world)
    torch.cuda.synchronize()
    ws.reset_counters()
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        my_ms = time_region(torch, step, args.steps, stream)
        barrier(world)
        torch.cuda.synchronize()
        wall_s = time.perf_counter() - t0
    clocks = clk.summary()
    cnt = ws.read_counters()  # layers decoded and kept channels in the timed region
    max_ms = max_over_ranks(my_ms, world, torch.device("cuda", local))
    value = whole_job_value(world, args.steps, max_ms)
    layer_calls = int(cnt["calls"])
    kept_per_layer = cnt["kept"] / max(layer_calls, 1)
    # one floe_v3::decode launch per token (every layer), or one fused launch per
    # layer when FLOE_MULTI=0
    multi = model.multi_layer
    launches = args.steps if multi else layer_calls
    # algorithmic bytes of one layer launch: f16 mixing + router +
    # 2 experts' up codes/meta + the kept records + the vectors
    layer_bytes = (MIX_BYTES + E * DH * 4 + TOPK * (CODE_BYTES + META_BYTES) +
                   kept_per_layer * REC_BYTES + 4 * 4 * DH)
    step_ms = my_ms / args.steps
    layer_us = step_ms * 1e3 / L
    achieved = layer_bytes / (layer_us * 1e-6) / 1e9

    # ---------------- per-launch duration without PDL overlap (stage profiling) ----
    ws.set_profiling(True)
    ws.read_profile()
    time_region(torch, step, min(args.steps, 4), stream)
    prof = ws.read_profile()
    ws.set_profiling(False)
    fused = prof.get("fused", {"ms": 0.0, "launches": 0})
    iso_us = 1e3 * fused["ms"] / max(fused["launches"], 1)
    # dram bytes per launch from the committed ncu --set full capture of the same
    # kernel (profiles/ncu_traffic.json, written by tools/summarize_ncu.py)
    traffic = None
    tf = ROOT / "profiles" / "ncu_traffic.json"
    kname = "decode" if multi else "fused"
    if tf.exists():
        traffic = json.loads(tf.read_text()).get(kname)
    per_launch = L if multi else 1
    roofline = {"bound": "hbm",
                "kernel": ("floe_v3::decode<4096> (every layer of the token in one launch)"
                           if multi else "floe_v2::fused<4096> (layer mode)"),
                "achieved": round(achieved, 1), "peak": hbm_peak, "peak_kind": peak_kind,
                "unit": "GB/s", "frac": round(achieved / hbm_peak, 4), "traffic": traffic,
                "traffic_source": f"profiles/ncu_traffic.json[{kname}] (ncu --set full, per launch)",
                "algorithmic_bytes_per_launch": int(layer_bytes * per_launch),
                "avg_launch_us": round(layer_us * per_launch, 3),
                "avg_launch_us_note": ("CUDA events over the timed region on the launching "
                                       "stream / launches"),
                "isolated_launch_us": round(iso_us, 3),
                "isolated_launch_note": "one launch alone (no programmatic dependent launch)"}

    # ---------------- config 1 (+ config-4 expert level) ----------------
    expert_ffn = run_expert(fb, torch, args, stream, hbm_peak)

    # ---------------- configs 4 and 5 at the layer level (C ABI) ----------------
    batched_layer = run_batched_layer(fb, torch, layers[0], ws, stream)

    # ---------------- e2e through the host-buffer C ABI ----------------
    # host buffers in page-locked memory (the serving process's I/O buffers):
    # the ABI copies them directly, no staging memcpy
    hs_h = hs.cpu().pin_memory().numpy()
    y_h = torch.empty((L, DH), dtype=torch.float32).pin_memory().numpy()
    for i in range(min(args.warmup, 3)):
        model.decode_host(hs_h[i], ws, out=y_h, replay=True)
    torch.cuda.synchronize()
    e2e_s = 0.0
    for i in range(args.steps):
        t1 = time.perf_counter()
        model.decode_host(hs_h[args.warmup + i], ws, out=y_h, replay=True)
        e2e_s += time.perf_counter() - t1
    e2e_max = max_over_ranks(e2e_s, world, torch.device("cuda", local))
    e2e = {"value": round(world * args.steps / e2e_max, 3), "unit": "tokens/s",
           "h2d_bytes_per_step": 4 * DH * L, "d2h_bytes_per_step": 4 * DH * L,
           "api": "floe_gpu_model_decode_host (replay: the token's 32 block inputs in, "
                  "32 block outputs back, from/to page-locked host buffers; stream sync)"}

    out = {
        "metric": METRIC, "value": round(value, 3), "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_ms, 5),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 accumulate (INT2 up codes, f16 gate/down records, f16 mixing)",
        "data": ("synthetic: reference gen_model streams (seed 7) generated+quantized on "
                 "device; block inputs token_input(1, 32 i + l) (replay)"),
        "config": {"workload": WORKLOAD, "layers": L, "d_hidden": DH, "d_intermediate": DI,
                   "experts": E, "top_k": TOPK, "bits": BITS, "group_size": G,
                   "sparsity_k": KSP,
                   "thresholds": ("calibrate_model(k=0.8) per layer on the device "
                                  f"({N_CAL} tokens token_input(3, t)), "
                                  f"mean {float(np.mean(thresholds)):.4f}"),
                   "kept_channels_per_layer": round(kept_per_layer, 1),
                   "parallelism": "replicas" if world > 1 else "single-gpu",
                   "l2": (f"inputs larger than L2: {L * 0.1645:.2f} GB of weights per token "
                          "(126 MB L2), no flush; K steps back to back in one event region")},
        "roofline": roofline,
        "layer": {"workload": "config2: the same layer launches (one Mixtral MoE layer, "
                              "single-token decode)",
                  "value": round(value * L, 1), "unit": "layer-tokens/s",
                  "us_per_layer": round(layer_us, 3),
                  "bytes_per_layer": int(layer_bytes)},
        "expert_ffn": expert_ffn,
        "batched_layer": batched_layer,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clocks,
        "wall_s_timed_region": round(wall_s, 4),
        "setup_s": round(setup_s, 2),
        "device": dev,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(thresholds, hs_h[args.warmup:], L)
    if not args.no_offload and world == 1:
        try:
            out["offload"] = run_offload(fb, torch, layers, ws, 6, 16.0, stream)
        except Exception as e:  # report, do not lose the main line
            out["offload"] = {"error": str(e)[:200]}
    if world > 1:
        dist.destroy_process_group()
    return out


def run_batched_layer(fb, torch, layer, ws, stream):
    """Configs 4 and 5 through floe_gpu_layer_forward_batched on layer 0 of the
    bench model: B decode tokens (config 4: B = 16, 64) and a 4,096-token
    prefill (config 5 on one GPU; device routing and dispatch, prefill GEMMs,
    tensor-core mixing).  Tokens token_input(1, 7000 + t)."""
    out = {}
    for B, key in ((16, "config4_b16"), (64, "config4_b64"), (EP_TOKENS, "config5_prefill")):
        H = torch.stack([fb.gen_normals(1, (1 << 40) + 7000 + t, DH) for t in range(B)])
        Y = torch.empty_like(H)
        for _ in range(2):
            fb.layer_forward_batched(layer, H, ws, out=Y)
        torch.cuda.synchronize()
        n = 5
        ms = time_region(torch, lambda i: fb.layer_forward_batched(layer, H, ws, out=Y), n, stream) / n
        out[key] = {"tokens": B, "ms_per_call": round(ms, 3), "value": round(B / (ms * 1e-3), 1),
                    "unit": "layer-tokens/s"}
    out["note"] = ("one Mixtral MoE layer, B tokens per call: <= 10 tokens go token by token "
                   "through the fused layer kernel; experts with >= 5 tokens through the prefill "
                   "path (exact tcgen05 up projection or dequantized f16 hi/lo GEMM, dense f16 "
                   "gate/down GEMMs); experts routed > 1 token run concurrently on 8 side "
                   "streams after their up projections")
    return out


def run_expert(fb, torch, args, stream, hbm_peak):
    """Config 1: seeded_expert(4096, 14336, 99 + j) for j < N_EXPERTS_C1 (cycled so that
    no step's 65 MB is L2-resident), seeded_input(4096, 100), INT2 g64,
    t_j = calibrate_threshold(|v_j|, 0.8), generated on the device."""
    sd = float(np.float32(1.0) / np.sqrt(np.float32(DH)))
    x = fb.gen_normals(100, 4, DH)
    ws = fb.Workspace(DH, DI, 1)
    exs, ths = [], []
    for j in range(N_EXPERTS_C1):
        gate = fb.gen_normals(99 + j, 1, DH * DI, sd)
        up = fb.gen_normals(99 + j, 2, DH * DI, sd)
        down = fb.gen_normals(99 + j, 3, DH * DI, sd)
        codes, scales, zeros = fb.quantize(up, BITS, G)
        del up
        ex = fb.GpuExpert(DH, DI, BITS, G, codes, scales, zeros, gate=gate, down=down)
        del gate, down
        v = fb.qgemv_channels(ex, x, ws)
        t = quantile_threshold(torch, v.abs(), KSP)
        ex.set_threshold(t)
        exs.append(ex)
        ths.append(t)
    y = torch.empty(DH, dtype=torch.float32, device="cuda")
    nk = torch.zeros(1, dtype=torch.int32, device="cuda")
    step = lambda i: fb.expert_forward_sparse(exs[i % N_EXPERTS_C1], x, ws, out=y, n_kept=nk)  # noqa: E731
    time_region(torch, step, args.warmup, stream)
    total_ms = time_region(torch, step, args.steps, stream)
    fb.expert_forward_sparse(exs[0], x, ws, out=y, n_kept=nk)
    n_kept = int(nk.item())
    ws.set_profiling(True)
    ws.read_profile()
    time_region(torch, step, args.steps, stream)
    prof = ws.read_profile()
    bytes_tok = CODE_BYTES + META_BYTES + n_kept * REC_BYTES + 8 * DH
    mean_ms = total_ms / args.steps
    gbs = bytes_tok / (mean_ms * 1e-3) / 1e9
    kernels = {}
    for k, p in prof.items():
        if p["launches"]:
            avg = p["ms"] / p["launches"]
            b = {"k1_up_threshold": CODE_BYTES + META_BYTES + 4 * DH,
                 "k2_gate_down": n_kept * REC_BYTES + 8 * DH, "fused": bytes_tok}.get(k)
            kernels[k] = {"avg_us": round(avg * 1e3, 3),
                          "gbs": round(b / (avg * 1e-3) / 1e9, 1) if b and avg > 0 else None}
    # config 4 (started): 16 tokens at once through the batched expert forward
    # (tcgen05 up projection + union gate/down) on the same experts
    B4 = 16
    X4 = torch.stack([fb.gen_normals(1, (1 << 40) + t, DH) for t in range(B4)])
    step4 = lambda i: fb.expert_forward_batched(exs[i % N_EXPERTS_C1], X4)  # noqa: E731
    n4 = max(4, args.steps // 8)
    time_region(torch, step4, 3, stream)
    ms4 = time_region(torch, step4, n4, stream) / n4
    batched = {"workload": "config4 (expert level): 16 tokens, batched expert_forward_sparse",
               "tokens": B4, "us_per_call": round(ms4 * 1e3, 2),
               "value": round(B4 / (ms4 * 1e-3), 1), "unit": "expert-tokens/s",
               "vs_batch1_value": round(B4 / (ms4 * 1e-3) / (1e3 / mean_ms), 3)}
    return {"workload": (f"config1: seeded_expert(4096,14336,99+j), j<{N_EXPERTS_C1} cycled, "
                         "seeded_input(4096,100), INT2 g64, k=0.8, batch 1"),
            "batched_16": batched,
            "value": round(1e3 / mean_ms, 1), "unit": "expert-tokens/s",
            "us_per_expert_token": round(mean_ms * 1e3, 3), "kept": n_kept,
            "threshold": round(ths[0], 6), "bytes_per_expert_token": bytes_tok,
            "achieved": round(gbs, 1), "peak": hbm_peak, "unit_bw": "GB/s",
            "frac": round(gbs / hbm_peak, 4),
            "kernels": kernels}


# ------------------------------------------------------------------ reference arm
REF_LAYERS = 2  # layers of the model the reference arm builds and times (a bounded sample)


def ref_model_from_thresholds(thresholds, workers):
    """gen_model(seed 7, REF_LAYERS layers) -> compress_model(INT2 g64, given
    thresholds) in the UNMODIFIED reference core (oracle/_ref/libfloe_ref.so)."""
    from oracle import oracle as O
    if O.REF is None:
        return None, None
    th = np.ascontiguousarray(np.asarray(thresholds, np.float32)[:REF_LAYERS].reshape(-1))
    cm = O.REF.ref_cmodel_build_thresholds(REF_LAYERS, E, TOPK, DH, DI, SEED, th, BITS, G,
                                           workers)
    if not cm:
        raise RuntimeError(O.ref_error())
    return O, cm


def cpu_baseline(thresholds, hs_h, L, budget_s=15.0):
    """Reference layer_forward(CompressedModel) on ONE host thread (the reference
    path is single-threaded) over a bounded sample: the first REF_LAYERS layers
    of the same model, the same thresholds and replayed block inputs; per-token
    time = L x the mean layer time (every layer has the same shapes)."""
    O, cm = ref_model_from_thresholds(thresholds, os.cpu_count() or 1)
    if cm is None:
        return {"value": None, "unit": "tokens/s", "cores": 1, "kind": "reference",
                "sample": "unavailable: oracle/_ref/libfloe_ref.so missing"}
    y = np.empty(DH, np.float32)
    t0 = time.perf_counter()
    O.REF.ref_layer_forward(cm, 0, np.ascontiguousarray(hs_h[0][0]), y)
    one = time.perf_counter() - t0
    n = int(min(max(budget_s / max(one, 1e-3), 2), 64))
    t0 = time.perf_counter()
    for i in range(n):
        tok, l = divmod(i, REF_LAYERS)
        O.REF.ref_layer_forward(cm, l, np.ascontiguousarray(hs_h[tok % len(hs_h)][l]), y)
    dt = time.perf_counter() - t0
    O.REF.ref_cmodel_destroy(cm)
    return {"value": round(n / dt / L, 5), "unit": "tokens/s", "cores": 1, "kind": "reference",
            "sample": (f"{n} floe::layer_forward calls over layers 0..{REF_LAYERS - 1} of the "
                       f"same model and inputs (1 thread, {dt:.1f} s); tokens/s = layer "
                       f"calls/s / {L}"), "cpu": cpu_model()}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip() + f" x{os.cpu_count()}"
    except OSError:
        pass
    return f"unknown x{os.cpu_count()}"



def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU path on all host threads, rank 0
    only: gen_model(seed 7) -> calibrate_model(k=0.8) per layer (as the GPU arm
    calibrates) -> compress_model -> layer_forward(CompressedModel) on replayed
    block inputs, independent (token, layer) calls split over the threads.  A
    bounded sample: REF_LAYERS of the 32 layers; tokens/s = layer calls/s / 32."""
    from oracle import oracle as O
    L = args.layers
    if O.REF is None:
        return {"impl": "reference", "metric": METRIC, "unit": "tokens/s",
                "unavailable": "oracle/_ref/libfloe_ref.so not built (reference sources absent)"}
    threads = os.cpu_count() or 1
    t_setup = time.perf_counter()
    ths = np.empty(REF_LAYERS * E, np.float32)
    cm = O.REF.ref_cmodel_build_replay(REF_LAYERS, E, TOPK, DH, DI, SEED, 3, N_CAL, KSP, BITS, G,
                                       threads, ths)
    if not cm:
        raise RuntimeError(O.ref_error())
    setup_s = time.perf_counter() - t_setup
    per_step = threads  # one layer call per thread per step
    n_calls = (args.warmup + args.steps) * per_step
    # replayed block inputs token_input(1, 32 i + l) of the same layers as the GPU arm
    toks = np.stack([O.token_input(1, L * (c // REF_LAYERS) + (c % REF_LAYERS), DH)
                     for c in range(min(n_calls, 4096))])
    toks = np.ascontiguousarray(np.resize(toks, (n_calls, DH)))
    times = []
    for s in range(args.warmup + args.steps):
        base = s * per_step
        dt = O.REF.ref_layer_calls_replicas(cm, REF_LAYERS, toks[base:base + per_step], per_step,
                                            threads)
        if dt < 0:
            raise RuntimeError("reference layer_forward failed")
        if s >= args.warmup:
            times.append(dt)
    O.REF.ref_cmodel_destroy(cm)
    total = sum(times)
    value = args.steps * per_step / total / L
    return {"impl": "reference", "metric": METRIC, "value": round(value, 5), "unit": "tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * total / args.steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic: reference gen_model (seed 7) + calibrate_model + compress_model, "
                    "host; replayed block inputs token_input(1, 32 i + l)",
            "config": {"workload": WORKLOAD, "layers": L, "d_hidden": DH, "d_intermediate": DI,
                       "experts": E, "top_k": TOPK, "bits": BITS, "group_size": G,
                       "sparsity_k": KSP,
                       "thresholds": (f"calibrate_model(k=0.8) per layer ({N_CAL} tokens), "
                                      f"mean {float(np.mean(ths)):.4f}"),
                       "parallelism": f"{threads} host threads, independent layer calls"},
            "cpu_baseline": {"value": round(value, 5), "unit": "tokens/s", "cores": threads,
                             "kind": "reference",
                             "sample": (f"{per_step} floe::layer_forward calls per step over "
                                        f"layers 0..{REF_LAYERS - 1} (one per thread); "
                                        f"tokens/s = layer calls/s / {L}"),
                             "cpu": cpu_model()},
            "e2e": {"value": round(value, 5), "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "setup_s": round(setup_s, 2)}


# ------------------------------------------------------------------ config 5 (--ep)
EP_TOKENS = 4096


def run_ep(args, rank, world, local):
    """Config 5: one expert-parallel MoE layer prefill of EP_TOKENS tokens, the 8
    experts sharded over the ranks (rank r owns experts [r E/W, (r+1) E/W)), each
    rank routing its EP_TOKENS/W tokens and exchanging them with all-to-alls
    (paper_2505_05950_b200/ep.py; NCCL over NVLink).  Strong scaling: the total
    is fixed.  --ep-cpu runs the same plumbing on CPU with gloo and a toy shape
    (tests/test_bench_multirank.py)."""
    import torch
    import torch.distributed as dist

    from paper_2505_05950_b200 import ep
    cpu = args.ep_cpu
    if world > 1:
        if cpu:
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    per = E // world
    first = rank * per
    if cpu:
        from oracle import oracle as O
        dh, di, T = 64, 32, 64
        rng = np.random.default_rng(5)
        ex = []
        for e in range(E):
            gate, up, down = O.seeded_expert(dh, di, 60 + e)
            ex.append(O.Expert(dh, di, O.quantize(up, 4, 16), gate, down, 0.3))
        router = torch.from_numpy((rng.standard_normal((E, dh)) / 8).astype(np.float32))
        mixing = torch.from_numpy((rng.standard_normal((dh, dh)) / 8).astype(np.float32))
        H = torch.from_numpy(np.stack([O.token_input(1, t, dh) for t in range(T)]))

        def expert_fn(e, X):
            Xn = X.numpy()
            return torch.from_numpy(np.stack([O.expert_forward_sparse(ex[e], x) for x in Xn])
                                    if len(Xn) else np.zeros((0, dh), np.float32))
        sync = lambda: None  # noqa: E731
        clock = time.perf_counter
    else:
        import paper_2505_05950_b200 as fb
        dh, T = DH, EP_TOKENS
        router, mixing, gate, up, down = gen_float_layer(fb, 0)
        th = calibrate_layer(fb, torch, router, mixing, gate, up, down)
        ex = []
        for e in range(first, first + per):
            codes, scales, zeros = fb.quantize(up[e].reshape(-1), BITS, G)
            ex.append(fb.GpuExpert(DH, DI, BITS, G, codes, scales, zeros, gate=gate[e],
                                   down=down[e], threshold=th[e]))
        del gate, up, down
        H = torch.stack([fb.gen_normals(1, (1 << 40) + 9000 + t, DH) for t in range(T)])
        mixing = mixing.half()  # the device layers' f16 mixing: tensor-core GEMMs
        expert_fn = ep.batched_expert_fn(ex, first_expert=first)
        sync = torch.cuda.synchronize
        clock = time.perf_counter
    lo, hi = T * rank // world, T * (rank + 1) // world

    def step():
        y, _, _ = ep.ep_moe_layer(H[lo:hi], router, mixing, TOPK, expert_fn, E)
        return y

    for _ in range(args.warmup):
        step()
    sync()
    barrier(world)
    t0 = clock()
    for _ in range(args.steps):
        step()
    sync()
    my_ms = (clock() - t0) * 1e3
    barrier(world)
    max_ms = my_ms
    if world > 1:
        t = torch.tensor([my_ms], dtype=torch.float64,
                         device="cpu" if cpu else torch.device("cuda", local))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        max_ms = float(t.item())
        dist.destroy_process_group()
    value = T * args.steps / (max_ms / 1000.0)
    return {"metric": "expert-parallel MoE layer prefill tokens/s (Mixtral-8x7B shape)",
            "value": round(value, 1), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(max_ms / args.steps, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32 accumulate (INT2 up codes, f16 gate/down records, f16 mixing; "
                     "f16 tensor-core GEMMs on hi/lo splits)",
            "data": "synthetic: gen_model layer 0 (seed 7), tokens token_input(1, 9000 + t)",
            "config": {"workload": (f"config5: one MoE layer prefill, {T} tokens, {E} experts "
                                    f"sharded over {world} rank(s), all-to-all dispatch/combine"),
                       "tokens": T, "d_hidden": dh, "experts": E, "top_k": TOPK,
                       "experts_per_rank": per,
                       "parallelism": f"ep{world}", "device": "cpu (gloo test)" if cpu else "cuda"}}


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--layers", type=int, default=N_MODEL_LAYERS)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-offload", action="store_true")
    ap.add_argument("--ep", action="store_true", help="config 5: expert-parallel layer prefill")
    ap.add_argument("--ep-cpu", action="store_true", help=argparse.SUPPRESS)  # gloo test mode
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank, world, local = dist_env()
    if args.ep or args.ep_cpu:
        out = run_ep(args, rank, world, local)
        if rank == 0:
            print(json.dumps(out), flush=True)
        return
    if args.impl == "reference":
        if rank != 0:
            return
        out = run_reference(args, rank, world)
        print(json.dumps(out), flush=True)
        return
    out = run_ours(args, rank, world, local)
    if rank == 0:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
