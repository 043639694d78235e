"""Config 1 through a CUDA graph: the host launch rate vs the kernel's own time."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import numpy as np  # noqa: E402


def main():
    import torch
    import paper_2505_05950_b200 as fb
    DH, DI = bench.DH, bench.DI
    sd = float(np.float32(1.0) / np.sqrt(np.float32(DH)))
    x = fb.gen_normals(100, 4, DH)
    ws = fb.Workspace(DH, DI, 1)
    exs = []
    for j in range(4):
        gate = fb.gen_normals(99 + j, 1, DH * DI, sd)
        up = fb.gen_normals(99 + j, 2, DH * DI, sd)
        down = fb.gen_normals(99 + j, 3, DH * DI, sd)
        codes, scales, zeros = fb.quantize(up, bench.BITS, bench.G)
        ex = fb.GpuExpert(DH, DI, bench.BITS, bench.G, codes, scales, zeros, gate=gate, down=down)
        v = fb.qgemv_channels(ex, x, ws)
        ex.set_threshold(bench.quantile_threshold(torch, v.abs(), bench.KSP))
        exs.append(ex)
    y = torch.empty(DH, device="cuda")
    st = torch.cuda.current_stream()
    step = lambda i: fb.expert_forward_sparse(exs[i % 4], x, ws, out=y)  # noqa: E731
    bench.time_region(torch, step, 8, st)
    ms = bench.time_region(torch, step, 200, st) / 200
    print(f"eager: {ms * 1e3:.2f} us/call")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(8):
            step(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(32):
            fb.expert_forward_sparse(exs[i % 4], x, ws, out=y, stream=s)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    msg = bench.time_region(torch, lambda i: g.replay(), 10, st) / (10 * 32)
    print(f"graph: {msg * 1e3:.2f} us/call")


if __name__ == "__main__":
    main()
