"""The multi-layer decode kernel (floe_v3::decode, one launch per token) against
the per-layer fused kernel (floe_v2::fused, one launch per layer) on the same
model and inputs: per-layer agreement and steady-state time per layer."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def main():
    import torch

    import paper_2505_05950_b200 as fb
    torch.cuda.set_device(0)
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    layers, _ = bench.build_model(fb, torch, L)
    model = fb.GpuModel(layers)
    ws = fb.Workspace(bench.DH, bench.DI, bench.TOPK)
    hs = bench.replay_inputs(fb, torch, 6, L)
    st = torch.cuda.current_stream()
    worst = 0.0
    for i in range(3):
        ym = model.decode(hs[i], ws, replay=True)
        torch.cuda.synchronize()
        yr = torch.stack([fb.layer_forward(layers[l], hs[i][l], ws) for l in range(L)])
        torch.cuda.synchronize()
        rel = ((ym - yr).norm(dim=1) / yr.norm(dim=1)).max().item()
        worst = max(worst, rel)
        print(f"token {i}: replay max rel-L2 over layers {rel:.3e}", flush=True)
    # chained
    # (the bench model's layers are not normalised: chained through more than
    # a few layers the activations overflow f32, so chain the first 3)
    LC = min(L, 3)
    model_c = fb.GpuModel(layers[:LC])
    yc = model_c.decode(hs[0][0], ws, replay=False)
    h = hs[0][0]
    for l in range(LC):
        h = fb.layer_forward(layers[l], h, ws)
    torch.cuda.synchronize()
    fin = torch.isfinite(h)
    same_nf = bool((torch.isfinite(yc) == fin).all())
    relc = ((yc[fin] - h[fin]).norm() / h[fin].norm().clamp_min(1e-30)).item() if same_nf else float("nan")
    print(f"chained: rel-L2 {relc:.3e} over {int(fin.sum())} finite of {h.numel()}", flush=True)
    # timing: steady state over 20 tokens
    ym = torch.empty(L, bench.DH, device="cuda")
    n = 20
    for i in range(3):
        model.decode(hs[i % 6], ws, out=ym, replay=True)
    ms = bench.time_region(torch, lambda i: model.decode(hs[i % 6], ws, out=ym, replay=True), n, st)
    ys = torch.empty(bench.DH, device="cuda")
    ms2 = bench.time_region(
        torch, lambda i: [fb.layer_forward(layers[l], hs[i % 6][l], ws, out=ys) for l in range(L)], n, st)
    print(f"multi: {ms * 1e3 / (n * L):.2f} us/layer   per-layer launches: {ms2 * 1e3 / (n * L):.2f} us/layer",
          flush=True)
    print("RESULT", "ok" if worst < 1e-2 and relc < 1e-3 else "MISMATCH")


if __name__ == "__main__":
    main()
