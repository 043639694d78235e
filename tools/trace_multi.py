"""Phase trace of one layer of the multi-layer decode kernel (floe_v3::decode) in
steady state: %globaltimer marks per CTA (FLOE_TRACE_LAYER, default 6 of 8),
printed as percentiles over CTAs relative to the first end-of-previous-layer
ticket."""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
os.environ.setdefault("FLOE_TRACE_LAYER", "6")
import bench  # noqa: E402

NAMES = [
    (29, "prev: ticket taken"), (20, "P prev: ticket seen"), (21, "P prev: chunk issued"),
    (30, "prev: layer barrier passed"), (22, "P prev: lpass seen"),
    (27, "P prev: h issued"), (11, "P: first item landed"), (15, "P: last prefetched landed"), (31, "P: layer top"), (23, "P: tail items issued"), (53, "P: last tail landed"),
    (0, "layer top"), (7, "h + slices in"), (8, "A batch 0 in"), (10, "A batch 1 in"),
    (12, "A batch 2 in"), (13, "A batch 3 in"), (39, "w0: pred published"), (38, "w8: start"),
    (40, "w8: batch 0"), (41, "w8: batch 1"), (42, "w8: batch 2"), (43, "w8: batch 3"),
    (44, "w9: batch 0"), (45, "w9: batch 1"), (46, "w9: batch 2"), (47, "w9: batch 3"), (14, "A items done"), (1, "phase A done"), (2, "routing barrier out"),
    (26, "R: predicted routing"), (24, "R: bar1 seen"), (25, "R: exact routing"),
    (16, "P: bar1 seen"), (35, "P: proxy fence done"), (32, "P: C->K1 ring free"), (33, "P: u issued"), (34, "u landed"), (17, "P: K1 tiles issued"), (3, "K1 setup done"), (4, "K1 done"),
    (18, "P: records start"), (5, "first record"), (19, "P: all issued"), (6, "C done"),
]


def main():
    import torch

    import paper_2505_05950_b200 as fb
    torch.cuda.set_device(0)
    L = 8
    layers, _ = bench.build_model(fb, torch, L)
    model = fb.GpuModel(layers)
    ws = fb.Workspace(bench.DH, bench.DI, bench.TOPK)
    hs = bench.replay_inputs(fb, torch, 6, L)
    ws.set_phase_trace(True)
    traces = []
    for i in range(6):
        model.decode(hs[i], ws, replay=True)
        torch.cuda.synchronize()
        T = ws.read_phase_trace().astype(np.int64)
        if i >= 1:
            traces.append(T)
    T = np.stack(traces)  # [steps, G, 96]
    t0 = np.where(T[:, :, 29] > 0, T[:, :, 29], np.iinfo(np.int64).max).min(axis=1)
    print(f"{len(traces)} steps, {T.shape[1]} CTAs; times in us from the first ticket of the previous layer")
    for m, nm in NAMES:
        v = T[:, :, m]
        ok = v > 0
        if not ok.any():
            continue
        rel = ((v - t0[:, None]) / 1e3)[ok]
        q = np.percentile(rel, [0, 10, 50, 90, 100])
        print(f"  {nm:28s} n={ok.sum():4d} min {q[0]:6.2f} p10 {q[1]:6.2f} med {q[2]:6.2f} "
              f"p90 {q[3]:6.2f} max {q[4]:6.2f}")
    span = (T[:, :, 6].max(1) - t0) / 1e3
    print(f"  previous ticket -> last C done: {span.mean():.2f} us")
    n = T[:, :, 9].ravel()
    print(f"  kept records per CTA: mean {n.mean():.1f} min {n.min()} max {n.max()}")
    by_ticket(T, t0)
    own = T[:, :, 28].ravel() < 128
    dA = ((T[:, :, 14] - T[:, :, 7]) / 1e3)  # h in -> A items done, per step and CTA
    ok = T[:, :, 14] > 0
    sm = T[:, :, 52]
    slow = ok & (dA > 9)
    print(f"  phase A (h->items done) per CTA: slow(>9us) fraction {slow.sum() / ok.sum():.2f}")
    for st in range(T.shape[0]):
        print("   step", st, "slow CTAs:", sorted(np.nonzero(slow[st])[0].tolist())[:40])
        print("          their SMs:", sorted(sm[st][slow[st]].tolist())[:40])


def by_ticket(T, t0):
    """Phase-A completion by the chunk owner's ticket (the chunk index)."""
    tau = T[:, :, 28]
    done = (T[:, :, 14] - t0[:, None]) / 1e3
    hin = (T[:, :, 7] - t0[:, None]) / 1e3
    tk = (T[:, :, 29] - t0[:, None]) / 1e3
    iss = (T[:, :, 21] - t0[:, None]) / 1e3
    lst = (T[:, :, 15] - t0[:, None]) / 1e3
    for lo in range(0, 148, 16):
        sel = (tau >= lo) & (tau < lo + 16) & (T[:, :, 14] > 0)
        if sel.any():
            print(f"  tickets {lo:3d}-{lo + 15:3d}: ticket at {tk[sel].mean():6.2f}  issued {iss[sel].mean():6.2f}"
                  f"  prefetch landed {lst[sel].mean():6.2f}  h in {hin[sel].mean():6.2f}"
                  f"  A items done {done[sel].mean():6.2f} (max {done[sel].max():6.2f})")


if __name__ == "__main__":
    main()
