"""Host submission cost per call vs device time per step (decides whether the
decode loop is launch-bound), and the same loop replayed from a CUDA graph."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402


def main():
    import torch

    import paper_2505_05950_b200 as fb
    from paper_2505_05950_b200 import _abi as A
    torch.cuda.set_device(0)
    ws = fb.Workspace(bench.DH, bench.DI, bench.TOPK)
    layers = []
    for li in range(4):
        r, m, ex = bench.build_layer(fb, torch, li)
        bench.calibrate(fb, torch, r, m, ex, ws)
        layers.append(fb.GpuLayer(r.cpu().numpy(), m.cpu().numpy(), ex, bench.TOPK, mixing_f16=True))
    toks = torch.stack([fb.gen_normals(1, (1 << 40) + t, bench.DH) for t in range(8)])
    y = torch.empty(bench.DH, device="cuda")
    st = torch.cuda.current_stream()
    N = 200
    for name, call in (
            ("python layer_forward", lambda i: fb.layer_forward(layers[i & 3], toks[i & 7], ws, out=y)),
            ("raw ctypes", lambda i, L=A.lib(), s=st.cuda_stream, hp=[t.data_ptr() for t in toks],
             yp=y.data_ptr(), lh=[l.handle for l in layers], wh=ws.handle:
             L.floe_gpu_layer_forward(lh[i & 3], wh, hp[i & 7], yp, None, s))):
        for i in range(10):
            call(i)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record(st)
        for i in range(N):
            call(i)
        t1 = time.perf_counter()
        b.record(st)
        torch.cuda.synchronize()
        print(f"{name:22s} host {1e6 * (t1 - t0) / N:7.2f} us/call   device {1e3 * a.elapsed_time(b) / N:7.2f} us/step")
    # the same loop captured once into a CUDA graph and replayed
    g = torch.cuda.CUDAGraph()
    s2 = torch.cuda.Stream()
    s2.wait_stream(st)
    with torch.cuda.stream(s2):
        for i in range(3):
            fb.layer_forward(layers[i & 3], toks[i & 7], ws, out=y, stream=s2.cuda_stream)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s2):
            for i in range(N):
                fb.layer_forward(layers[i & 3], toks[i & 7], ws, out=y, stream=s2.cuda_stream)
    st.wait_stream(s2)
    g.replay()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(st)
    g.replay()
    b.record(st)
    torch.cuda.synchronize()
    print(f"{'cuda graph replay':22s} device {1e3 * a.elapsed_time(b) / N:7.2f} us/step")


if __name__ == "__main__":
    main()
