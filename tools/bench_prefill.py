"""Prefill expert forward (floe_gpu_expert_forward_prefill) on a Mixtral expert:
time per call and tensor-core throughput against the batched path."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402


def main():
    import torch

    import paper_2505_05950_b200 as fb
    n_el = bench.DH * bench.DI
    gate = fb.gen_normals(99, 1, n_el, 1.0 / 64.0)
    up = fb.gen_normals(99, 2, n_el, 1.0 / 64.0)
    down = fb.gen_normals(99, 3, n_el, 1.0 / 64.0)
    codes, scales, zeros = fb.quantize(up, bench.BITS, bench.G)
    e = fb.GpuExpert(bench.DH, bench.DI, bench.BITS, bench.G, codes, scales, zeros, gate=gate,
                     down=down, threshold=1.0)
    st = torch.cuda.current_stream()
    for n in (4, 8, 16, 32, 64, 96, 256, 1024, 2048):
        X = torch.stack([fb.gen_normals(1, (1 << 40) + t, bench.DH) for t in range(n)])
        Y = torch.empty_like(X)
        for _ in range(2):
            fb.expert_forward_prefill(e, X, out=Y)
        torch.cuda.synchronize()
        k = 5
        ms = bench.time_region(torch, lambda i: fb.expert_forward_prefill(e, X, out=Y), k, st) / k
        flops = 2.0 * n * bench.DH * bench.DI * 5  # K1 (K = 3 dh) + gate + down GEMMs
        out = {"tokens": n, "ms": round(ms, 3), "tflops": round(flops / (ms * 1e-3) / 1e12, 1)}
        if n <= 64 and n >= 16:
            msb = bench.time_region(torch, lambda i: fb.expert_forward_batched(e, X), k, st) / k
            out["batched_ms"] = round(msb, 3)
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
