"""Short driver for ncu captures: builds the bench workload (one Mixtral MoE
layer + the config-1 expert) and runs a few flushed decode steps of each.

    ncu --set full -k regex:'k1_int2|k2_gate_down|mixing_route' -s 6 -c 3 \
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
    ap.add_argument("--what", choices=["layer", "expert", "both"], default="both")
    args = ap.parse_args()
    import torch

    import paper_2505_05950_b200 as fb
    torch.cuda.set_device(0)
    flush = torch.zeros(64 << 20, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    if args.what in ("layer", "both"):
        router, mixing, experts = bench.build_layer(fb, torch)
        ws = fb.Workspace(bench.DH, bench.DI, bench.TOPK)
        bench.calibrate(fb, torch, router, mixing, experts, ws)
        layer = fb.GpuLayer(router.cpu().numpy(), mixing.cpu().numpy(), experts, bench.TOPK)
        toks = torch.stack([fb.gen_normals(1, (1 << 40) + t, bench.DH) for t in range(args.steps)])
        y = torch.empty(bench.DH, device="cuda")
        torch.cuda.synchronize()
        print("PROFILE-LAYER-START", flush=True)
        bench.time_steps(torch, lambda i: fb.layer_forward(layer, toks[i], ws, out=y),
                         args.steps, flush, stream)
    if args.what in ("expert", "both"):
        a = argparse.Namespace(steps=args.steps, warmup=1)
        print(bench.run_expert(fb, torch, a, flush, stream, 6549.4))


if __name__ == "__main__":
    main()
