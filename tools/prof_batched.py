"""One batched tcgen05 up-projection call (B tokens) on a Mixtral expert, for ncu."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402


def main():
    import torch

    import paper_2505_05950_b200 as fb
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    up = fb.gen_normals(99, 2, bench.DH * bench.DI, 1.0 / 64.0)
    codes, scales, zeros = fb.quantize(up, bench.BITS, bench.G)
    e = fb.GpuExpert(bench.DH, bench.DI, bench.BITS, bench.G, codes, scales, zeros)
    X = torch.stack([fb.gen_normals(1, (1 << 40) + t, bench.DH) for t in range(B)])
    for _ in range(3):
        fb.qgemv_channels_batched(e, X)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
