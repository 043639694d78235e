"""One config-4 batched layer call (B tokens) for an ncu launch list
(ncu --profile-from-start off: only the second call is captured).
    python tools/prof_blayer.py B [nows]   (nows: no workspace, so small
    batches take the batched path instead of the per-token kernel)"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def main():
    import torch

    import paper_2505_05950_b200 as fb
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    torch.cuda.set_device(0)
    layers, _ = bench.build_model(fb, torch, 1)
    ws = None if (len(sys.argv) > 2 and sys.argv[2] == "nows") else fb.Workspace(bench.DH, bench.DI, bench.TOPK)
    H = torch.stack([fb.gen_normals(1, (1 << 40) + 7000 + t, bench.DH) for t in range(B)])
    fb.layer_forward_batched(layers[0], H, ws)
    torch.cuda.synchronize()
    print("PROFILE-START", flush=True)
    torch.cuda.profiler.start()
    fb.layer_forward_batched(layers[0], H, ws)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()


if __name__ == "__main__":
    main()
