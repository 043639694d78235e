"""Per-phase timing of the fused kernel via in-kernel %globaltimer marks
(floe_v2.cuh mark()): distribution over CTAs of each interval, averaged over
several flushed steps, for layer mode and single-expert mode."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402

# consumer marks: 0 start, 1 phase A done, 6 barrier-1 passed, 2 routed, 7 first K1
# tile landed, 3 K1 done, 8 published, 4 barrier-2 passed, 9 plan done, 10 first
# record landed, 11 first pool record landed, 5 phase C done.
# producer marks: 16 K1 issue start, 17 prefetch issued, 18 plan seen, 19 own
# issued, 20 all issued.
LAYER = [(0, 1, "A mixing"), (1, 6, "grid barrier 1"), (6, 2, "route"),
         (2, 7, "first K1 tile lands"), (7, 3, "K1 tiles"), (3, 8, "publish"),
         (8, 4, "grid barrier 2"), (4, 9, "plan"), (9, 10, "first record"),
         (10, 11, "own records"), (11, 5, "pool records"), (16, 17, "P: K1 issue+prefetch"),
         (18, 19, "P: own issue"), (19, 20, "P: pool issue")]
EXPERT = [(0, 2, "start -> K1")] + LAYER[3:]


def summarize(tag, traces, marks):
    T = np.stack(traces).astype(np.int64)  # [steps, G, 64]
    t0 = T[:, :, 0].min(axis=1)
    print(f"== {tag}: {T.shape[0]} steps, {T.shape[1]} CTAs")
    for (a, b, name) in marks:
        ok = (T[:, :, a] > 0) & (T[:, :, b] > 0)
        if not ok.any():
            continue
        d = ((T[:, :, b] - T[:, :, a]) / 1e3)[ok]
        print(f"   {name:24s} mean {d.mean():7.2f}  min {d.min():7.2f}  max {d.max():7.2f} us")
    end = (T[:, :, 5].max(1) - t0) / 1e3
    print(f"   first start -> last phase-C end: {end.mean():7.2f} us")
    names = {0: "start", 1: "A done", 6: "barrier1 out", 12: "partials (w0)", 13: "partials (all)",
             14: "top-k done", 15: "softmax done",
             2: "routed", 7: "1st tile", 3: "K1 done",
             8: "published", 18: "P: all published", 5: "C done"}
    for m, nm in names.items():
        v = T[:, :, m]
        if not (v > 0).any():
            continue
        rel = (v - t0[:, None]) / 1e3
        rel = rel[v > 0]
        q = np.percentile(rel, [0, 10, 50, 90, 100])
        print(f"   t[{nm:16s}] min {q[0]:6.2f} p10 {q[1]:6.2f} med {q[2]:6.2f} p90 {q[3]:6.2f} max {q[4]:6.2f}")


def main():
    import torch

    import paper_2505_05950_b200 as fb
    torch.cuda.set_device(0)
    ws = fb.Workspace(bench.DH, bench.DI, bench.TOPK)
    layers, experts0 = [], []
    for li in range(bench.N_LAYERS):  # distinct layers cycled: nothing L2-resident
        router, mixing, experts = bench.build_layer(fb, torch, li)
        bench.calibrate(fb, torch, router, mixing, experts, ws)
        layers.append(fb.GpuLayer(router.cpu().numpy(), mixing.cpu().numpy(), experts,
                                  bench.TOPK))
        experts0.append(experts[0])
    toks = torch.stack([fb.gen_normals(1, (1 << 40) + t, bench.DH) for t in range(12)])
    y = torch.empty(bench.DH, device="cuda")
    ws1 = fb.Workspace(bench.DH, bench.DI, 1)
    for name, w, run, marks in (
            ("layer", ws, lambda i: fb.layer_forward(layers[i % 4], toks[i], ws, out=y), LAYER),
            ("expert", ws1, lambda i: fb.expert_forward_sparse(experts0[i % 4], toks[i], ws1,
                                                               out=y), EXPERT)):
        w.set_phase_trace(True)
        traces = []
        for i in range(12):
            run(i)
            torch.cuda.synchronize()
            if i >= 2:
                traces.append(w.read_phase_trace())
            else:
                w.read_phase_trace()
        summarize(name, traces, marks)
        T = np.stack(traces).astype(np.int64)
        if name == "layer":
            d0 = (T[:, :, 65] - T[:, :, 13]) / 1e3
            print("   back-to-back marks histogram (us):", np.histogram(d0, bins=[0, 0.5, 1, 1.5, 2, 3, 4, 6, 10])[0].tolist())
            d = (T[:, :, 14] - T[:, :, 65]) / 1e3
            print("   top-k interval histogram (us):", np.histogram(d, bins=[0, 0.5, 1, 1.5, 2, 3, 4, 6, 10])[0].tolist())
            cdone = (T[-1, :, 5] - T[-1, :, 0].min()) / 1e3
            order = np.argsort(cdone)[::-1][:8]
            print("   slowest phase-C CTAs (cta, C done us, own, deficit, P, plan->done us):",
                  [(int(c), round(float(cdone[c]), 1), int(T[-1, c, 66]), int(T[-1, c, 67]),
                    int(T[-1, c, 68]), round(float((T[-1, c, 5] - T[-1, c, 9]) / 1e3), 1)) for c in order])
            so = T[:, :, 71]
            if (so > 0).any():
                print("   speculation: ok", int((so == 2).sum()), "mispredicted", int((so == 1).sum()))
            print("   own+deficit spread:", int((T[-1, :, 66] + T[-1, :, 67]).min()), int((T[-1, :, 66] + T[-1, :, 67]).max()))
            smid = T[-1, :, 64]
            slow = d[-1] > 1.5
            print("   slow CTAs' SMs (last step):", sorted(smid[slow].tolist()))
            print("   fast CTAs' SMs (last step):", sorted(smid[~slow].tolist())[:60])
            for st in range(T.shape[0]):
                print("   step", st, "slow count", int((d[st] > 1.5).sum()), "slow SMs even/odd:",
                      int((smid[d[st] > 1.5] % 2 == 0).sum()), int((smid[d[st] > 1.5] % 2 == 1).sum()))
        for cta in (0, 37, 100):
            tr = T[-1, cta]
            base = tr[48]
            iss = [(tr[48 + k] - base) / 1e3 for k in range(16) if tr[48 + k]]
            bat = [tuple((tr[24 + 4 * i + j] - base) / 1e3 for j in range(4)) for i in range(6)
                   if tr[24 + 4 * i]]
            print(f"   CTA {cta}: issue " + " ".join(f"{v:.1f}" for v in iss))
            print("          batches (start,ready,barrier,done) " +
                  " ".join("(" + ",".join(f"{x:.2f}" for x in b4) + ")" for b4 in bat))


if __name__ == "__main__":
    main()



def slow_ctas(T, a, b, thr_us=1.5):
    """CTAs whose interval a->b exceeds thr_us in the last trace, with %smid."""
    d = (T[-1, :, b] - T[-1, :, a]) / 1e3
    return [(int(i), round(float(d[i]), 2)) for i in np.nonzero(d > thr_us)[0]]
