"""Experiment: step time of the layer / expert under different L2 conditions.

  dirty : flush by writing a 256 MiB buffer (leaves ~126 MB of dirty lines)
  clean : flush by reading a 256 MiB buffer (L2 full of clean lines)
  none  : back-to-back steps (weights partly L2-resident from the last step)
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def main():
    import torch

    import paper_2505_05950_b200 as fb
    torch.cuda.set_device(0)
    router, mixing, experts = bench.build_layer(fb, torch)
    ws = fb.Workspace(bench.DH, bench.DI, bench.TOPK)
    bench.calibrate(fb, torch, router, mixing, experts, ws)
    layer = fb.GpuLayer(router.cpu().numpy(), mixing.cpu().numpy(), experts, bench.TOPK)
    n = 40
    toks = torch.stack([fb.gen_normals(1, (1 << 40) + t, bench.DH) for t in range(n)])
    y = torch.empty(bench.DH, device="cuda")
    buf = torch.zeros(64 << 20, dtype=torch.float32, device="cuda")
    sink = torch.zeros(1, device="cuda")
    stream = torch.cuda.current_stream()

    def run(mode, fn):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(n)]
        for i in range(n):
            if mode == "dirty":
                buf.add_(1.0)
            elif mode == "clean":
                sink.copy_(buf.sum())
            evs[i][0].record(stream)
            fn(i)
            evs[i][1].record(stream)
        torch.cuda.synchronize()
        ms = sorted(a.elapsed_time(b) for a, b in evs)[5:-5]
        return sum(ms) / len(ms) * 1e3

    layer_fn = lambda i: fb.layer_forward(layer, toks[i], ws, out=y)  # noqa: E731
    ex = experts[0]
    ws1 = fb.Workspace(bench.DH, bench.DI, 1)
    x = toks[0]
    exp_fn = lambda i: fb.expert_forward_sparse(ex, toks[i], ws1, out=y)  # noqa: E731
    for mode in ("dirty", "clean", "none"):
        run(mode, layer_fn)
        print(f"layer  {mode:6s} {run(mode, layer_fn):8.2f} us")
        run(mode, exp_fn)
        print(f"expert {mode:6s} {run(mode, exp_fn):8.2f} us")
    # per-stage with clean flush
    ws.set_profiling(True)
    ws.read_profile()
    run("clean", layer_fn)
    print({k: round(v["ms"] * 1e3 / max(v["launches"], 1), 2) for k, v in ws.read_profile().items()})
    del x


if __name__ == "__main__":
    main()
