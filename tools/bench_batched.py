"""Throughput of the batched up projection (config 4's K1: the IMMA kernel up
to 16 tokens, the tcgen05 kernel above) on a
Mixtral-shaped expert: one pass over the 18.35 MB of codes+meta for B tokens.
Prints per-B time, tokens/s and achieved HBM GB/s of the algorithmic bytes
(codes + meta + x + v), 4 distinct experts cycled (inputs > L2).

    python tools/bench_batched.py [--iters 50]
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def forward(fb, torch, args, hbm_peak):
    """Batched expert_forward_sparse: K1 on tcgen05 + union gate/down, vs B
    single-token fused calls on the same experts and tokens."""
    sd = float(1.0 / 64.0)
    exs, ths = [], []
    x0 = fb.gen_normals(100, 4, bench.DH)
    ws = fb.Workspace(bench.DH, bench.DI, 1)
    for j in range(4):
        gate = fb.gen_normals(99 + j, 1, bench.DH * bench.DI, sd)
        up = fb.gen_normals(99 + j, 2, bench.DH * bench.DI, sd)
        down = fb.gen_normals(99 + j, 3, bench.DH * bench.DI, sd)
        codes, scales, zeros = fb.quantize(up, bench.BITS, bench.G)
        e = fb.GpuExpert(bench.DH, bench.DI, bench.BITS, bench.G, codes, scales, zeros, gate=gate,
                         down=down)
        th = bench.quantile_threshold(torch, fb.qgemv_channels(e, x0, ws).abs(), bench.KSP)
        e.set_threshold(th)
        exs.append(e)
        ths.append(th)
        del gate, up, down
    lines = []
    for B in (1, 4, 16, 32, 64):
        X = torch.stack([fb.gen_normals(1, (1 << 40) + t, bench.DH) for t in range(B)])
        V = torch.empty((B, bench.DI), device="cuda")
        fb.expert_forward_batched(exs[0], X, v=V)
        union = int((V.abs() >= ths[0]).any(0).sum())
        for i in range(3):
            fb.expert_forward_batched(exs[i % 4], X)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(args.iters):
            fb.expert_forward_batched(exs[i % 4], X)
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) * 1e3 / args.iters
        # the same tokens one by one through the single-token fused kernel
        a.record()
        for i in range(max(1, args.iters // 4)):
            for t in range(B):
                fb.expert_forward_sparse(exs[i % 4], X[t], ws)
        b.record()
        torch.cuda.synchronize()
        us1 = a.elapsed_time(b) * 1e3 / max(1, args.iters // 4)
        byts = bench.CODE_BYTES + bench.META_BYTES + union * bench.REC_BYTES + 8 * B * bench.DH
        d = {"workload": "config4 expert: batched expert_forward_sparse, one Mixtral expert, k=0.8",
             "tokens": B, "union_channels": union, "us_per_call": round(us, 2),
             "token_expert_per_s": round(B / (us * 1e-6), 1),
             "single_token_path_us_for_B": round(us1, 2), "speedup_vs_single": round(us1 / us, 2),
             "bytes": byts, "gbs": round(byts / (us * 1e-6) / 1e9, 1), "hbm_peak_gbs": hbm_peak,
             "frac": round(byts / (us * 1e-6) / 1e9 / hbm_peak, 4)}
        print(json.dumps(d), flush=True)
        lines.append(d)
    return lines


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--out", default=None)
    ap.add_argument("--forward", action="store_true", help="batched expert forward (K1 + gate/down)")
    args = ap.parse_args()
    import torch

    import paper_2505_05950_b200 as fb
    torch.cuda.set_device(0)
    hbm_peak, _ = bench.peaks()
    if args.forward:
        lines = forward(fb, torch, args, hbm_peak)
        if args.out:
            Path(args.out).write_text("\n".join(json.dumps(d) for d in lines) + "\n")
        return
    sd = float(1.0 / 64.0)
    exs = []
    for j in range(8):
        up = fb.gen_normals(99 + j, 2, bench.DH * bench.DI, sd)
        codes, scales, zeros = fb.quantize(up, bench.BITS, bench.G)
        exs.append(fb.GpuExpert(bench.DH, bench.DI, bench.BITS, bench.G, codes, scales, zeros))
        del up
    lines = []
    for B in (1, 4, 8, 16, 32, 64):
        X = torch.stack([fb.gen_normals(1, (1 << 40) + t, bench.DH) for t in range(B)])
        for i in range(5):
            fb.qgemv_channels_batched(exs[i % len(exs)], X)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(args.iters):
            fb.qgemv_channels_batched(exs[i % len(exs)], X)
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) * 1e3 / args.iters
        byts = bench.CODE_BYTES + bench.META_BYTES + 4 * B * (bench.DH + bench.DI)
        d = {"workload": "config4 K1: batched up projection, one Mixtral expert (4096x14336 INT2 g64)",
             "tokens": B, "us_per_call": round(us, 2), "token_expert_per_s": round(B / (us * 1e-6), 1),
             "bytes": byts, "gbs": round(byts / (us * 1e-6) / 1e9, 1), "hbm_peak_gbs": hbm_peak,
             "frac": round(byts / (us * 1e-6) / 1e9 / hbm_peak, 4),
             "kernel": "floe_k1b::k1 (IMMA)" if B <= 16 else "floe_tc::k1_batched (tcgen05)",
             "note": "includes the per-call token prep kernels and stream-ordered scratch alloc"}
        print(json.dumps(d), flush=True)
        lines.append(d)
    if args.out:
        Path(args.out).write_text("\n".join(json.dumps(d) for d in lines) + "\n")


if __name__ == "__main__":
    main()
