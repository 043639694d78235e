"""Throughput of the tcgen05 batched up projection (config 4's K1) on a
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch

    import paper_2505_05950_b200 as fb
    torch.cuda.set_device(0)
    hbm_peak, _ = bench.peaks()
    sd = float(1.0 / 64.0)
    exs = []
    for j in range(8):
        up = fb.gen_normals(99 + j, 2, bench.DH * bench.DI, sd)
        codes, scales, zeros = fb.quantize(up, bench.BITS, bench.G)
        exs.append(fb.GpuExpert(bench.DH, bench.DI, bench.BITS, bench.G, codes, scales, zeros))
        del up
    lines = []
    for B in (1, 4, 16, 32, 64):
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
             "note": "includes the per-call token prep kernels and stream-ordered scratch alloc"}
        print(json.dumps(d), flush=True)
        lines.append(d)
    if args.out:
        Path(args.out).write_text("\n".join(json.dumps(d) for d in lines) + "\n")


if __name__ == "__main__":
    main()
