"""Profiling workload for the multi-layer decode kernel (floe_v3::decode): an
L-layer model (argv[1], default 8), `steps` replay decodes (ncu -k regex:decode -s 2 -c 1)."""
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
    hs = bench.replay_inputs(fb, torch, 4, L)
    for i in range(4):
        model.decode(hs[i], ws, replay=True)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
