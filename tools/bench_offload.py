"""Config 3: Mixtral-shaped decode with every expert's gate|down
records host-resident (pinned host memory, read in place over PCIe by the
fused kernel), an LRU of whole experts in HBM under a VRAM budget.

    python tools/bench_offload.py [--layers 32] [--tokens 48] [--budgets-gb 0,16,1000]

Prints one JSON line per budget: decode tokens/s, bytes per token over PCIe,
achieved PCIe GB/s against the measured pinned host->device copy peak.
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def h2d_peak(torch):
    src = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
    dst = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
    best = 0.0
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dst.copy_(src, non_blocking=True)
        b.record()
        torch.cuda.synchronize()
        best = max(best, (1 << 30) / (a.elapsed_time(b) * 1e-3) / 1e9)
    del src, dst
    return best


def build(fb, torch, n_layers, host_records=True):
    sigma = float(np.float32(1.0) / np.sqrt(np.float32(bench.DH)))
    ws = fb.Workspace(bench.DH, bench.DI, bench.TOPK)
    layers = []
    for li in range(n_layers):
        router = fb.gen_normals(bench.SEED, bench.weight_stream(li, 0, 0), bench.E * bench.DH, sigma, sharded=True)
        mixing = fb.gen_normals(bench.SEED, bench.weight_stream(li, 1, 0), bench.DH * bench.DH, sigma, sharded=True)
        experts = []
        for e in range(bench.E):
            gate = fb.gen_normals(bench.SEED, bench.weight_stream(li, 2, e), bench.DH * bench.DI, sigma, sharded=True)
            up = fb.gen_normals(bench.SEED, bench.weight_stream(li, 3, e), bench.DH * bench.DI, sigma, sharded=True)
            down = fb.gen_normals(bench.SEED, bench.weight_stream(li, 4, e), bench.DH * bench.DI, sigma, sharded=True)
            codes, scales, zeros = fb.quantize(up, bench.BITS, bench.G)
            del up
            experts.append(fb.GpuExpert(bench.DH, bench.DI, bench.BITS, bench.G, codes, scales, zeros,
                                        gate=gate, down=down, threshold=0.0, host_records=host_records))
            del gate, down, codes, scales, zeros
        bench.calibrate(fb, torch, router, mixing.view(bench.DH, bench.DH), experts, ws)
        layers.append(fb.GpuLayer(router.view(bench.E, bench.DH).cpu().numpy(),
                                  mixing.view(bench.DH, bench.DH).cpu().numpy(), experts, bench.TOPK))
        torch.cuda.synchronize()
    return layers, ws


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--tokens", type=int, default=48)
    ap.add_argument("--warmup", type=int, default=48)
    ap.add_argument("--budgets-gb", default="0,16,1000")
    ap.add_argument("--out", default=None, help="append the JSON lines to this file")
    ap.add_argument("--dump-after", type=float, default=3600.0, help="dump Python stacks after N s")
    args = ap.parse_args()
    import faulthandler
    faulthandler.dump_traceback_later(args.dump_after, exit=False)
    import torch

    import paper_2505_05950_b200 as fb
    torch.cuda.set_device(0)
    peak = h2d_peak(torch)
    hbm_peak, _ = bench.peaks()
    t0 = time.perf_counter()
    layers, ws = build(fb, torch, args.layers)
    setup = time.perf_counter() - t0
    n = args.warmup + args.tokens
    # per token, one recorded block input per layer (decode_replay): every
    # layer sees N(0, 1) inputs like its calibration tokens, so it runs at the
    # calibrated sparsity (a chained random-weight stack without norms grows
    # its activations layer over layer and soon keeps every channel)
    L = args.layers
    toks = torch.stack([torch.stack([fb.gen_normals(1, (1 << 40) + t * L + l, bench.DH)
                                     for l in range(L)]) for t in range(n)])
    y = torch.empty(L, bench.DH, device="cuda")
    for gb in [float(x) for x in args.budgets_gb.split(",")]:
        off = fb.Offload(layers, int(gb * (1 << 30)))
        for t in range(args.warmup):
            off.decode_replay(toks[t], ws, out=y)
            torch.cuda.synchronize()
        s0 = off.stats()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for t in range(args.warmup, n):
            off.decode_replay(toks[t], ws, out=y)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        s1 = off.stats()
        rb = s1["record_bytes"]
        pcie = (s1["records_over_pcie"] - s0["records_over_pcie"]) * rb / args.tokens
        hbm = (s1["records_from_hbm"] - s0["records_from_hbm"]) * rb / args.tokens
        promoted = (s1["bytes_promoted"] - s0["bytes_promoted"]) / args.tokens
        tok_s = args.tokens / (ms * 1e-3)
        gbs = (pcie + promoted) / (ms * 1e-3 / args.tokens) / 1e9
        # HBM side: per layer the mixing matrix, router, both experts' up codes
        # and metadata, activations (bench.py's stage bytes), plus the kept
        # records of resident experts
        fixed = args.layers * (bench.MIX_BYTES + 3 * 4 * bench.DH + bench.E * bench.DH * 4 + 4 * bench.DH
                               + bench.TOPK * (bench.CODE_BYTES + bench.META_BYTES) + 4 * bench.DH
                               + 2 * 4 * bench.DH)
        hbm_gbs = (fixed + hbm) / (ms * 1e-3 / args.tokens) / 1e9
        line = json.dumps({
            "workload": f"config3: {args.layers}-layer Mixtral-8x7B-shaped decode, records host-resident",
            "vram_budget_gb": gb, "tokens": args.tokens, "tokens_per_s": round(tok_s, 2),
            "ms_per_token": round(ms / args.tokens, 3),
            "record_bytes_per_token_over_pcie": int(pcie), "record_bytes_per_token_from_hbm": int(hbm),
            "promoted_bytes_per_token": int(promoted),
            "pcie_gbs": round(gbs, 2), "pcie_peak_gbs": round(peak, 2),
            "pcie_frac": round(gbs / peak, 4),
            "hbm_bytes_per_token": int(fixed + hbm), "hbm_gbs": round(hbm_gbs, 1),
            "hbm_peak_gbs": hbm_peak, "hbm_frac": round(hbm_gbs / hbm_peak, 4),
            "promotions": s1["promotions"], "evictions": s1["evictions"],
            "device_record_gb": round(s1["device_record_bytes"] / (1 << 30), 2),
            "setup_s": round(setup, 1)})
        print(line, flush=True)
        if args.out:
            with open(args.out, "a") as f:
                f.write(line + "\n")
        off.close()


if __name__ == "__main__":
    main()
