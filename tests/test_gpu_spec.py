"""Predicted routing in the fused layer kernel: the producer streams the K1
tiles of the experts predicted by router_pred * h (router_pred = router +
router * mixing) during the mixing GEMV, and the consumers run K1 on them
before the exact routing of u exists; the prediction is verified before any
record is read.  The result must not depend on the prediction: a correct
prediction and a forced misprediction (FLOE_TEST_MISPREDICT=1 inverts the
predicted logits, so the re-run path executes) give the same routing, masks
and outputs, and those match the oracle (model.cpp:145-208)."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu

SHAPES = [(4096, 2048, 8, 2), (2048, 512, 8, 2), (2048, 1024, 16, 4)]


def _layer(dh, di, E, K):
    rng = np.random.default_rng(dh + di + E)
    experts = []
    for e in range(E):
        gate, up, down = O.seeded_expert(dh, di, 500 + e)
        q = O.quantize(up, 2, 64)
        experts.append(O.Expert(dh, di, q, gate, down, 0.0))
    router = (rng.standard_normal((E, dh)) / np.sqrt(dh)).astype(np.float32)
    mixing = (rng.standard_normal((dh, dh)) / np.sqrt(dh)).astype(np.float32)
    # per-expert thresholds: 0.8-quantile of |v| on one calibration token
    u = O.token_input(3, 0, dh)
    u = u + mixing @ u
    for ex in experts:
        ex.threshold = O.calibrate_threshold(np.abs(O.qgemv_channels(ex.up_q, dh, u)), 0.8)
    return O.Layer(router, mixing, experts, K)


def _run(out_path):
    """Run every shape's layer over a few tokens; save the traced results."""
    import torch

    import paper_2505_05950_b200 as fb
    res = {}
    for si, (dh, di, E, K) in enumerate(SHAPES):
        L = _layer(dh, di, E, K)
        ex = [fb.GpuExpert(dh, di, 2, 64, e.up_q.codes, e.up_q.scales, e.up_q.zeros, gate=e.gate,
                           down=e.down_t, threshold=e.threshold) for e in L.experts]
        gl = fb.GpuLayer(L.router, L.mixing, ex, K, mixing_f16=True)
        ws = fb.Workspace(dh, di, K)
        for t in range(4):
            h = torch.from_numpy(O.token_input(1, t, dh)).cuda()
            tr = fb.layer_forward(gl, h, ws, traced=True)
            torch.cuda.synchronize()
            for k in ("experts", "weights", "masks", "out"):
                res[f"{si}_{t}_{k}"] = tr[k].cpu().numpy()
    np.savez(out_path, **res)


def _subprocess(tmp_path, name, env_extra):
    out = tmp_path / f"{name}.npz"
    env = dict(os.environ, **env_extra)
    code = f"import sys; sys.path.insert(0, {str(ROOT / 'tests')!r}); import test_gpu_spec as t; t._run({str(out)!r})"
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return dict(np.load(out))


def test_speculation_never_changes_results(tmp_path):
    spec = _subprocess(tmp_path, "spec", {"FLOE_TEST_MISPREDICT": "0"})
    miss = _subprocess(tmp_path, "miss", {"FLOE_TEST_MISPREDICT": "1"})
    for key in spec:
        for other in (miss,):
            if key.endswith("_out"):
                assert O.rel_l2(other[key], spec[key]) <= 1e-6, key
            else:
                assert np.array_equal(other[key], spec[key]), key


def test_speculative_layer_matches_oracle(tmp_path):
    spec = _subprocess(tmp_path, "spec2", {"FLOE_TEST_MISPREDICT": "0"})
    for si, (dh, di, E, K) in enumerate(SHAPES):
        L = _layer(dh, di, E, K)
        L.mixing = L.mixing.astype(np.float16).astype(np.float32)  # the device reads f16 mixing
        for t in range(4):
            ref = O.layer_forward(L, O.token_input(1, t, dh), traced=True)
            assert np.array_equal(spec[f"{si}_{t}_experts"], ref["experts"].astype(np.int32))
            m, rm = spec[f"{si}_{t}_masks"], ref["masks"]
            diff = np.nonzero(m != rm)
            assert len(diff[0]) <= 16, len(diff[0])
            assert O.rel_l2(spec[f"{si}_{t}_out"], ref["out"]) <= 1e-2
