"""Handle lifetimes and descriptor propagation (round-1 advisor findings):

* a layer copies its experts' descriptors into a device table; destroying the
  layer must unregister that table, so a later residency change of a borrowed
  expert does not write into freed memory, and the expert keeps working in a
  new layer;
* set_threshold after layer (and model) creation must reach layer_forward and
  the multi-layer decode, not only expert_forward_sparse (the threshold table
  is per expert, model.cpp:237).
"""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

DH, DI, E, K = 2048, 256, 8, 2


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available()
    return torch


@pytest.fixture(scope="module")
def fb(torch):
    import paper_2505_05950_b200 as fb
    return fb


def _parts(seed):
    rng = np.random.default_rng(seed)
    oex = []
    for j in range(E):
        gate, up, down = O.seeded_expert(DH, DI, seed + j)
        q = O.quantize(up, 2, 64)
        t = O.calibrate_threshold(np.abs(O.qgemv_channels(q, DH, O.seeded_input(DH, 5))), 0.8)
        oex.append(O.Expert(DH, DI, q, gate, down, t))
    router = (rng.standard_normal((E, DH)) / np.sqrt(DH)).astype(np.float32)
    mixing = (rng.standard_normal((DH, DH)) / np.sqrt(DH) / 4).astype(np.float32)
    return oex, router, mixing


def _gpu_experts(fb, oex):
    return [fb.GpuExpert(DH, DI, 2, 64, e.up_q.codes, e.up_q.scales, e.up_q.zeros, gate=e.gate,
                         down=e.down_t, threshold=e.threshold) for e in oex]


def test_layer_destroyed_then_residency_change(fb, torch):
    oex, router, mixing = _parts(300)
    exs = _gpu_experts(fb, oex)
    ws = fb.Workspace(DH, DI, K)
    h = torch.from_numpy(O.token_input(1, 3, DH)).cuda()
    layer = fb.GpuLayer(router, mixing, exs, K)
    y0 = fb.layer_forward(layer, h, ws).cpu().numpy()
    layer.close()
    # the closed layer's table is no longer registered with the experts
    for e in exs:
        e.set_resident(False)
        e.set_resident(True)
    torch.cuda.synchronize()
    layer2 = fb.GpuLayer(router, mixing, exs, K)
    y1 = fb.layer_forward(layer2, h, ws).cpu().numpy()
    assert O.rel_l2(y1, y0) <= 1e-5
    ref = O.layer_forward(O.Layer(router, mixing, oex, K), O.token_input(1, 3, DH))
    assert O.rel_l2(y1, ref) <= 1e-2


def test_set_threshold_reaches_layer_and_model(fb, torch):
    oex, router, mixing = _parts(400)
    exs = _gpu_experts(fb, oex)
    ws = fb.Workspace(DH, DI, K)
    layer = fb.GpuLayer(router, mixing, exs, K, mixing_f16=True)
    model = fb.GpuModel([layer])
    x = O.token_input(1, 9, DH)
    h = torch.from_numpy(x).cuda()
    # keep every channel: threshold 0 (model.cpp:135 keeps |v| >= 0)
    for e, o in zip(exs, oex):
        e.set_threshold(0.0)
        o.threshold = 0.0
    y_layer = fb.layer_forward(layer, h, ws).cpu().numpy()
    y_model = model.decode(h, ws).cpu().numpy()
    mix16 = mixing.astype(np.float16).astype(np.float32)
    ref = O.layer_forward(O.Layer(router, mix16, oex, K), x)
    assert O.rel_l2(y_layer, ref) <= 1e-2
    assert O.rel_l2(y_model, ref) <= 1e-2
    # and the traced masks keep every channel of the routed experts
    tr = fb.layer_forward(layer, h, ws, traced=True)
    assert int(tr["masks"].sum().item()) == K * DI
