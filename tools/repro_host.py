"""Repro: device-path layer calls followed by host-buffer calls on one workspace."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402


def main():
    import torch

    import paper_2505_05950_b200 as fb
    torch.cuda.set_device(0)
    ws = fb.Workspace(bench.DH, bench.DI, bench.TOPK)
    r, m, ex = bench.build_layer(fb, torch, 0)
    bench.calibrate(fb, torch, r, m, ex, ws)
    layer = fb.GpuLayer(r.cpu().numpy(), m.cpu().numpy(), ex, bench.TOPK, mixing_f16=True)
    toks = torch.stack([fb.gen_normals(1, (1 << 40) + t, bench.DH) for t in range(8)])
    y = torch.empty(bench.DH, device="cuda")
    for i in range(4):
        fb.layer_forward(layer, toks[i], ws, out=y)
    torch.cuda.synchronize()
    print("device calls ok", flush=True)
    th = toks.cpu().numpy()
    yh = np.empty(bench.DH, np.float32)
    for i in range(4):
        fb.layer_forward_host(layer, th[i], ws, out=yh)
        print("host call ok", i, float(np.abs(yh).sum()), flush=True)


if __name__ == "__main__":
    main()
