"""Config 4/5 at the layer level: floe_gpu_layer_forward_batched over B tokens
(one Mixtral layer, device-calibrated thresholds, f16 mixing) against the same
tokens through the single-token fused layer kernel.  Prints JSON lines."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def main():
    import torch

    import paper_2505_05950_b200 as fb
    torch.cuda.set_device(0)
    st = torch.cuda.current_stream()
    layers, _ = bench.build_model(fb, torch, 2)
    ws = fb.Workspace(bench.DH, bench.DI, bench.TOPK)
    Bs = [int(b) for b in sys.argv[1].split(",")] if len(sys.argv) > 1 else (1, 4, 16, 64, 256, 1024, 4096)
    for B in Bs:
        H = torch.stack([fb.gen_normals(1, (1 << 40) + 7000 + t, bench.DH) for t in range(B)])
        fb.layer_forward_batched(layers[0], H)
        torch.cuda.synchronize()
        n = 3 if B >= 1024 else 6
        ms = bench.time_region(torch, lambda i: fb.layer_forward_batched(layers[i % 2], H), n, st) / n
        ys = torch.empty(bench.DH, device="cuda")
        nt = min(B, 64)
        ms1 = bench.time_region(torch, lambda i: fb.layer_forward(layers[i % 2], H[i % B], ws, out=ys),
                                nt, st) / nt
        print(json.dumps({"tokens": B, "batched_ms": round(ms, 3),
                          "batched_tok_s": round(B / (ms * 1e-3), 1),
                          "per_token_fused_tok_s": round(1 / (ms1 * 1e-3), 1)}), flush=True)


if __name__ == "__main__":
    main()
