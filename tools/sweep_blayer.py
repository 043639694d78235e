"""Batched-layer switch sweep: floe_gpu_layer_forward_batched WITH a workspace
(the bench's call) over token counts; run under different FLOE_* switches.
Prints one JSON line per token count."""
import json
import os
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
    env = {k: v for k, v in os.environ.items() if k.startswith("FLOE_")}
    for B in [int(b) for b in sys.argv[1].split(",")]:
        H = torch.stack([fb.gen_normals(1, (1 << 40) + 7000 + t, bench.DH) for t in range(B)])
        fb.layer_forward_batched(layers[0], H, ws)
        torch.cuda.synchronize()
        n = 8
        ms = bench.time_region(torch, lambda i: fb.layer_forward_batched(layers[i % 2], H, ws), n, st) / n
        print(json.dumps({"env": env, "tokens": B, "ms": round(ms, 3),
                          "tok_s": round(B / (ms * 1e-3), 1)}), flush=True)


if __name__ == "__main__":
    main()
