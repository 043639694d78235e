"""Is the phase-C time of a CTA a property of its SM?  Runs the layer step
several times with the phase trace and correlates per-SM phase-C durations
(plan known -> phase C done) across steps."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def main():
    import torch

    import paper_2505_05950_b200 as fb
    torch.cuda.set_device(0)
    ws = fb.Workspace(bench.DH, bench.DI, bench.TOPK)
    layers = []
    for li in range(2):
        r, m, ex = bench.build_layer(fb, torch, li)
        bench.calibrate(fb, torch, r, m, ex, ws)
        layers.append(fb.GpuLayer(r.cpu().numpy(), m.cpu().numpy(), ex, bench.TOPK, mixing_f16=True))
    ws.set_phase_trace(True)
    per_sm = []
    for step in range(24):
        h = fb.gen_normals(1, (1 << 40) + step, bench.DH)
        fb.layer_forward(layers[step % 2], h, ws)
        torch.cuda.synchronize()
        T = np.asarray(ws.read_phase_trace(), dtype=np.int64)  # [G][slots]
        smid = T[:, 64]
        dur = (T[:, 5] - T[:, 9]) / 1e3
        d = np.full(148, np.nan)
        d[smid] = dur
        per_sm.append(d)
    P = np.stack(per_sm[4:])  # skip warm-up
    z = (P - P.mean(1, keepdims=True)) / P.std(1, keepdims=True)
    c = np.corrcoef(z)
    off = c[~np.eye(len(c), dtype=bool)]
    print("phase-C duration per SM: mean over steps of the per-step spread (max-min) us:",
          round(float(np.mean(P.max(1) - P.min(1))), 2))
    print("correlation of per-SM durations between steps: mean", round(float(off.mean()), 3),
          "min", round(float(off.min()), 3))
    slow = np.argsort(np.nanmean(z, 0))[-10:]
    print("consistently slow SMs:", slow.tolist(), np.round(np.nanmean(z, 0)[slow], 2).tolist())


if __name__ == "__main__":
    main()
