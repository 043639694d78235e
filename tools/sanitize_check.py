"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck):
the fused kernel in expert and layer mode (fast path), the generic kernels,
the batched tcgen05 up projection and batched expert forward, the prefill
path, and the multi-layer decode kernel.  Run with
FLOE_LIB=tools/libfloe_b200_sanitize.so (600 s barrier watchdog)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import oracle as O  # noqa: E402


def main():
    import torch

    import paper_2505_05950_b200 as fb
    torch.cuda.set_device(0)
    # expert mode, fast path
    dh, di = 2048, 512
    gate, up, down = O.seeded_expert(dh, di, 5)
    q = O.quantize(up, 2, 64)
    x = O.seeded_input(dh, 6)
    t = O.calibrate_threshold(np.abs(O.qgemv_channels(q, dh, x)), 0.8)
    e = fb.GpuExpert(dh, di, 2, 64, q.codes, q.scales, q.zeros, gate=gate, down=down, threshold=t)
    ws = fb.Workspace(dh, di, 2)
    y = fb.expert_forward_sparse(e, torch.from_numpy(x).cuda(), ws).cpu().numpy()
    assert np.isfinite(y).all()  # (parity is the tests' job; this exercises the kernels)
    # layer mode, fast path
    ex = [e]
    for i in range(3):
        qi = O.quantize(O.seeded_expert(dh, di, 7 + i)[1], 2, 64)
        ex.append(fb.GpuExpert(dh, di, 2, 64, qi.codes, qi.scales, qi.zeros, gate=gate, down=down,
                               threshold=t))
    rng = np.random.default_rng(1)
    layer = fb.GpuLayer((rng.standard_normal((4, dh)) / 45).astype(np.float32),
                        (rng.standard_normal((dh, dh)) / 45).astype(np.float32), ex, 2)
    for tok in range(2):
        fb.layer_forward(layer, torch.from_numpy(O.token_input(1, tok, dh)).cuda(), ws, traced=True)
    # generic path
    g2, u2, d2 = O.seeded_expert(64, 256, 3)
    q2 = O.quantize(u2, 8, 64)
    e2 = fb.GpuExpert(64, 256, 8, 64, q2.codes, q2.scales, q2.zeros, gate=g2, down=d2, threshold=0.5)
    ws2 = fb.Workspace(64, 256)
    fb.expert_forward_sparse(e2, torch.from_numpy(O.seeded_input(64, 4)).cuda(), ws2)
    # batched tcgen05 up projection and batched forward (ragged d_intermediate)
    gate3, up3, down3 = O.seeded_expert(2048, 520, 11)
    q3 = O.quantize(up3, 2, 64)
    e3 = fb.GpuExpert(2048, 520, 2, 64, q3.codes, q3.scales, q3.zeros, gate=gate3, down=down3,
                      threshold=1.0)
    X = torch.from_numpy(np.stack([O.token_input(1, i, 2048) for i in range(5)])).cuda()
    fb.qgemv_channels_batched(e3, X)
    fb.expert_forward_batched(e3, X)
    fb.expert_forward_batched(e3, X[:3])  # <= 4 tokens: the fused union kernel
    # the prefill path (exact batched K1 at 5 tokens; dequantized GEMM at 80)
    fb.expert_forward_prefill(e3, X)
    X80 = torch.from_numpy(np.stack([O.token_input(1, 100 + i, 2048) for i in range(80)])).cuda()
    fb.expert_forward_prefill(e3, X80)
    # the multi-layer decode kernel: 3 layers (f16 mixing), replay and chained,
    # two tokens (the second layer boundary takes the finish-order chunks)
    layers3 = []
    for li in range(3):
        exs = []
        for j in range(4):
            gj, uj, dj = O.seeded_expert(dh, di, 40 + 4 * li + j)
            qj = O.quantize(uj, 2, 64)
            exs.append(fb.GpuExpert(dh, di, 2, 64, qj.codes, qj.scales, qj.zeros, gate=gj, down=dj,
                                    threshold=t))
        layers3.append(fb.GpuLayer((rng.standard_normal((4, dh)) / 45).astype(np.float32),
                                   (rng.standard_normal((dh, dh)) / 45).astype(np.float32), exs, 2,
                                   mixing_f16=True))
    model = fb.GpuModel(layers3)
    assert model.multi_layer
    hs = torch.from_numpy(np.stack([O.token_input(1, 50 + i, dh) for i in range(3)])).cuda()
    for _ in range(2):
        model.decode(hs, ws, replay=True)
    model.decode(hs[0], ws)
    torch.cuda.synchronize()
    print("sanitize workload ok")


if __name__ == "__main__":
    main()
