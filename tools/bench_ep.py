"""Config 5 (expert-parallel prefill), one GPU: a Mixtral-shaped MoE layer
(d=4096, ffn=14336, 8 experts, top-2, INT2 g64, k=0.8) over 4096 prefill
tokens through paper_2505_05950_b200.ep (mixing/router GEMMs in torch, experts
through the batched expert forward in 64-token chunks).  Prints tokens/s."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def main():
    import torch

    import paper_2505_05950_b200 as fb
    from paper_2505_05950_b200 import ep
    torch.cuda.set_device(0)
    T = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    ws = fb.Workspace(bench.DH, bench.DI, bench.TOPK)
    router, mixing, experts = bench.build_layer(fb, torch, 0)
    bench.calibrate(fb, torch, router, mixing.view(bench.DH, bench.DH), experts, ws)
    R = router.view(bench.E, bench.DH)
    M = mixing.view(bench.DH, bench.DH)
    H = torch.stack([fb.gen_normals(1, (1 << 40) + t, bench.DH) for t in range(T)])
    fn = ep.batched_expert_fn(experts)
    ep.ep_moe_layer(H[:256], R, M, bench.TOPK, fn, bench.E)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    ep.ep_moe_layer(H, R, M, bench.TOPK, fn, bench.E)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    print(json.dumps({"workload": f"config5: {T}-token prefill, one Mixtral MoE layer, experts "
                      "through the batched expert forward (64-token chunks), 1 GPU",
                      "tokens": T, "ms": round(ms, 2), "tokens_per_s": round(T / (ms * 1e-3), 1),
                      "note": "expert-parallel over N GPUs shards the experts (paper_2505_05950_b200/ep.py); "
                              "measured here at N=1"}))


if __name__ == "__main__":
    main()
