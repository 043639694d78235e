"""Per-phase timing of the fused kernel via in-kernel %globaltimer marks
(floe_v2.cuh mark()): distribution over CTAs of each interval, averaged over
several flushed steps, for layer mode and single-expert mode."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402

# consumer marks (thread 0): 0 start, 1 phase A done (partials written),
# 2 grid barrier passed, 3 K1 setup done, 4 K1 done (list final), 5 first
# record consumed, 6 phase C done.  producer marks: 16 predicted routing seen
# (mixing issued), 17 K1 tiles issued, 18 record issue starts (routing
# verified), 19 all records issued.  router marks: 24 barrier seen, 25 routed.
LAYER = [(0, 7, "predicted partial"), (0, 26, "P: predicted routing"), (0, 8, "first mixing stage"), (0, 1, "A mixing"), (1, 2, "grid barrier"), (2, 3, "K1 setup"), (3, 4, "K1"),
         (4, 5, "first record"), (5, 6, "records"), (24, 25, "P: exact routing"),
         (16, 17, "P: K1 tile issue"), (17, 18, "P: wait routing"), (18, 19, "P: record issue"),
         (4, 27, "K1 done -> plan known")]
EXPERT = [(0, 3, "start -> K1")] + LAYER[6:9] + LAYER[11:]


def summarize(tag, traces, marks):
    T = np.stack(traces).astype(np.int64)  # [steps, G, slots]
    t0 = T[:, :, 0].min(axis=1)
    print(f"== {tag}: {T.shape[0]} steps, {T.shape[1]} CTAs")
    for (a, b, name) in marks:
        ok = (T[:, :, a] > 0) & (T[:, :, b] > 0)
        if not ok.any():
            continue
        d = ((T[:, :, b] - T[:, :, a]) / 1e3)[ok]
        print(f"   {name:24s} mean {d.mean():7.2f}  min {d.min():7.2f}  max {d.max():7.2f} us")
    end = (T[:, :, 6].max(1) - t0) / 1e3
    print(f"   first start -> last phase-C end: {end.mean():7.2f} us")
    names = {0: "start", 11: "pdl released", 7: "predicted", 8: "1st mixing", 1: "A done", 2: "barrier out", 25: "routed", 3: "K1 start",
             4: "K1 done", 5: "1st record", 6: "C done", 16: "P: predicted", 17: "P: tiles issued",
             18: "P: records start", 29: "published", 30: "R: all seen", 27: "R: plan known", 19: "P: all issued"}
    for m, nm in names.items():
        v = T[:, :, m]
        if not (v > 0).any():
            continue
        rel = (v - t0[:, None]) / 1e3
        rel = rel[v > 0]
        q = np.percentile(rel, [0, 10, 50, 90, 100])
        print(f"   t[{nm:17s}] min {q[0]:6.2f} p10 {q[1]:6.2f} med {q[2]:6.2f} p90 {q[3]:6.2f} max {q[4]:6.2f}")


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
            # steady state: 32-layer replay decode back to back (PDL), the trace
            # of the last launch
            layers32, _ = bench.build_model(fb, torch, 8)
            model = fb.GpuModel(layers32)
            hs = bench.replay_inputs(fb, torch, 4, 8)
            ysd = torch.empty(8, bench.DH, device="cuda")
            steady = []
            for i in range(4):
                model.decode(hs[i], ws, out=ysd, replay=True)
                torch.cuda.synchronize()
                steady.append(w.read_phase_trace())
            summarize("layer (steady state: last of 8 back-to-back launches)", steady, LAYER)
        for w in (0, 1, 4):
            sl = [T[:, :, 32 + w * 4 + k].mean() / 1e3 for k in range(4)]
            print(f"   K1 warp {w}: wait_full {sl[0]:.2f} compute {sl[1]:.2f} qbar {sl[2]:.2f} epilogue/other {sl[3]:.2f} us")
        n = T[:, :, 9].ravel()
        m = T[:, :, 28].ravel()
        if m.any():
            print(f"   processed records per CTA: mean {m.mean():.1f} min {m.min()} max {m.max()} sd {m.std():.1f}")
        d = ((T[:, :, 6] - T[:, :, 5]) / 1e3).ravel()
        print(f"   kept records per CTA: mean {n.mean():.1f} min {n.min()} max {n.max()} sd {n.std():.1f};"
              f" corr(records, phase-C time) {np.corrcoef(n, d)[0, 1]:.2f};"
              f" us/record {np.sum(d) / max(1, np.sum(n)):.3f}")


if __name__ == "__main__":
    main()

