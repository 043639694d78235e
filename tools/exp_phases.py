"""Per-phase timing of the fused kernel via in-kernel %globaltimer marks.

Prints, for layer mode and single-expert mode, the distribution over CTAs of
each phase's duration (us) and the launch skew, averaged over several steps.
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def summarize(tag, traces, marks):
    # traces: list of [G, 8] arrays
    T = np.stack(traces).astype(np.int64)  # [steps, G, 8]
    t0 = T[:, :, 0].min(axis=1, keepdims=True)
    print(f"== {tag}: {T.shape[0]} steps, {T.shape[1]} CTAs")
    print(f"   launch skew (max start - min start): {np.mean(T[:, :, 0].max(1) - T[:, :, 0].min(1)) / 1e3:7.2f} us")
    for (a, b, name) in marks:
        d = (T[:, :, b] - T[:, :, a]) / 1e3
        print(f"   {name:28s} mean {d.mean():7.2f}  min {d.min():7.2f}  max {d.max():7.2f} us")
    end = (T[:, :, 5].max(1) - t0[:, 0]) / 1e3
    print(f"   first start -> last phase-C end: {end.mean():7.2f} us")
    # phase-C record arrivals (after each wait) relative to phase-C start, CTA 0 and 100
    for cta in (0, 100):
        arr = T[-1, cta, 8:]
        base = T[-1, cta, 4]
        rel = [(x - base) / 1e3 for x in arr if x > base]
        print(f"   CTA {cta:3d} phase-C record arrivals (us): " +
              " ".join(f"{v:.1f}" for v in rel[:40]))


def main():
    import torch

    import paper_2505_05950_b200 as fb
    torch.cuda.set_device(0)
    flush = torch.zeros(64 << 20, dtype=torch.float32, device="cuda")
    sink = torch.zeros(1, device="cuda")
    router, mixing, experts = bench.build_layer(fb, torch)
    ws = fb.Workspace(bench.DH, bench.DI, bench.TOPK)
    bench.calibrate(fb, torch, router, mixing, experts, ws)
    layer = fb.GpuLayer(router.cpu().numpy(), mixing.cpu().numpy(), experts, bench.TOPK)
    toks = torch.stack([fb.gen_normals(1, (1 << 40) + t, bench.DH) for t in range(12)])
    y = torch.empty(bench.DH, device="cuda")
    ws.set_phase_trace(True)
    traces = []
    for i in range(12):
        sink.copy_(flush.sum())
        fb.layer_forward(layer, toks[i], ws, out=y)
        torch.cuda.synchronize()
        if i >= 2:
            traces.append(ws.read_phase_trace())
    summarize("layer (clean L2)", traces,
              [(0, 1, "A mixing"), (1, 2, "barrier1 + route"), (2, 3, "B K1 (2 experts)"),
               (3, 4, "barrier2"), (4, 5, "C K2")])
    ws1 = fb.Workspace(bench.DH, bench.DI, 1)
    ws1.set_phase_trace(True)
    traces = []
    for i in range(12):
        sink.copy_(flush.sum())
        fb.expert_forward_sparse(experts[0], toks[i], ws1, out=y)
        torch.cuda.synchronize()
        if i >= 2:
            traces.append(ws1.read_phase_trace())
    summarize("expert (clean L2)", traces,
              [(0, 2, "start -> K1"), (2, 3, "B K1"), (3, 4, "barrier2"), (4, 5, "C K2")])


if __name__ == "__main__":
    main()
