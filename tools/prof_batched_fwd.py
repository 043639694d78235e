"""Batched expert forward (config 4) on a Mixtral expert, B tokens, for ncu:
the tcgen05 K1 (k1_batched) plus the gate/down GEMMs (gate_gemm, down_gemm;
FLOE_GATE_TC=1 FLOE_DOWN_TC=1 force them at any B)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402


def main():
    import torch

    import paper_2505_05950_b200 as fb
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    n = bench.DH * bench.DI
    gate = fb.gen_normals(99, 1, n, 1.0 / 64.0)
    up = fb.gen_normals(99, 2, n, 1.0 / 64.0)
    down = fb.gen_normals(99, 3, n, 1.0 / 64.0)
    codes, scales, zeros = fb.quantize(up, bench.BITS, bench.G)
    e = fb.GpuExpert(bench.DH, bench.DI, bench.BITS, bench.G, codes, scales, zeros, gate=gate,
                     down=down, threshold=1.0)
    X = torch.stack([fb.gen_normals(1, (1 << 40) + t, bench.DH) for t in range(B)])
    for _ in range(3):
        fb.expert_forward_batched(e, X)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
