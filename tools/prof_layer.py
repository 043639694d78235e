"""Short driver for ncu captures of the fused kernel: one Mixtral MoE layer
(64 calibration launches of the K1-only mode come first), then --steps decode
steps; or the config-1 expert.

    ncu --set full --import-source on -k regex:fused -s 66 -c 1 \
        -o gpurun_out/prof python tools/prof_layer.py --steps 4
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--what", choices=["layer", "expert"], default="layer")
    args = ap.parse_args()
    import torch

    import paper_2505_05950_b200 as fb
    torch.cuda.set_device(0)
    stream = torch.cuda.current_stream()
    if args.what == "layer":
        router, mixing, experts = bench.build_layer(fb, torch)
        ws = fb.Workspace(bench.DH, bench.DI, bench.TOPK)
        bench.calibrate(fb, torch, router, mixing, experts, ws)  # 64 K1-only launches
        layer = fb.GpuLayer(router.cpu().numpy(), mixing.cpu().numpy(), experts, bench.TOPK)
        toks = torch.stack([fb.gen_normals(1, (1 << 40) + t, bench.DH) for t in range(args.steps)])
        y = torch.empty(bench.DH, device="cuda")
        torch.cuda.synchronize()
        print("PROFILE-LAYER-START", flush=True)
        bench.time_region(torch, lambda i: fb.layer_forward(layer, toks[i], ws, out=y),
                          args.steps, stream)
    else:
        a = argparse.Namespace(steps=args.steps, warmup=1)
        print(bench.run_expert(fb, torch, a, stream, 6547.2))


if __name__ == "__main__":
    main()
