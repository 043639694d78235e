"""The multi-layer decode kernel (floe_v3::decode): a token through every layer
of a model in ONE launch, the reference's `run` loop h = layer_forward(m, l, h)
(tools/cli.cpp:86-107; each layer core/src/model.cpp:145-208).

* against the reference core, layer by layer, on a 32-layer stack with f16
  mixing (replayed block inputs, predictor.cpp:60-85) and a chained 4-layer
  decode;
* against the per-layer fused kernel (floe_v2::fused) on the same layers: the
  two paths differ only in the order of the mixing dot products;
* the misprediction path (FLOE_TEST_MISPREDICT=1 inverts the predicted
  logits) gives the same outputs as the predicted path;
* Mixtral shape (d 4096, ffn 14336), the bench's own layers, against the
  per-layer kernel.
"""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tests"))
from test_gpu_parity_bench import _ref_stack, _upload_stack  # noqa: E402

pytestmark = pytest.mark.gpu

L, E_, K_, DH, DI = 32, 8, 2, 2048, 512


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available()
    return torch


@pytest.fixture(scope="module")
def fb(torch):
    import paper_2505_05950_b200 as fb
    return fb


@pytest.fixture(scope="module")
def stack(fb, ref):
    cm, _ = _ref_stack(ref, L, E_, K_, DH, DI)
    layers, keep = _upload_stack(fb, ref, cm, L, E_, K_, DH, DI, mixing_f16=True)
    yield cm, layers
    ref.ref_cmodel_destroy(cm)


def _replay(tok):
    return np.stack([O.token_input(1, L * tok + l, DH) for l in range(L)])


def test_stack_replay_vs_reference_core(fb, torch, ref, stack):
    cm, layers = stack
    model = fb.GpuModel(layers)
    assert model.multi_layer
    ws = fb.Workspace(DH, DI, K_)
    errs = []
    for tok in range(3):
        hs = _replay(tok)
        want = np.empty_like(hs)
        for l in range(L):
            assert ref.ref_layer_forward(cm, l, hs[l], want[l]) == 0
        got = model.decode(torch.from_numpy(hs).cuda(), ws, replay=True).cpu().numpy()
        errs += [O.rel_l2(got[l], want[l]) for l in range(L)]
    errs = np.array(errs)
    # f16 mixing against the reference's f32: a routing near-tie may flip one layer
    assert np.sum(errs > 1e-2) <= 2, np.sort(errs)[-5:]
    assert float(np.median(errs)) <= 2e-3, float(np.median(errs))


def test_stack_vs_per_layer_kernel(fb, torch, stack):
    _, layers = stack
    model = fb.GpuModel(layers)
    ws = fb.Workspace(DH, DI, K_)
    errs = []
    for tok in range(3):
        hs = torch.from_numpy(_replay(tok)).cuda()
        got = model.decode(hs, ws, replay=True)
        want = torch.stack([fb.layer_forward(layers[l], hs[l], ws) for l in range(L)])
        errs += [O.rel_l2(got[l].cpu().numpy(), want[l].cpu().numpy()) for l in range(L)]
    errs = np.array(errs)
    # same arithmetic except the mixing sums' order: a channel within an ulp of
    # its threshold may flip
    assert float(np.median(errs)) <= 1e-5, float(np.median(errs))
    assert errs.max() <= 2e-2, errs.max()


def test_chained_decode(fb, torch, ref, stack):
    cm, layers = stack
    ws = fb.Workspace(DH, DI, K_)
    h0 = O.token_input(1, 999, DH)
    h = h0.copy()
    for l in range(4):
        y = np.empty_like(h)
        assert ref.ref_layer_forward(cm, l, h, y) == 0
        h = y
    model4 = fb.GpuModel(layers[:4])
    assert model4.multi_layer
    got = model4.decode(torch.from_numpy(h0).cuda(), ws).cpu().numpy()
    assert O.rel_l2(got, h) <= 1e-2
    # host-buffer entry point (pinned staging) gives the device result, up to the
    # order of the y additions (red.add from every CTA)
    got_h = model4.decode_host(h0, ws)
    assert O.rel_l2(got_h, got) <= 1e-5
    # page-locked caller buffers are copied directly (no staging memcpy)
    h_pin = torch.from_numpy(h0).pin_memory()
    y_pin = torch.empty(DH, dtype=torch.float32).pin_memory()
    model4.decode_host(h_pin.numpy(), ws, out=y_pin.numpy())
    assert O.rel_l2(y_pin.numpy(), got) <= 1e-5


def _mispredict_run(out_path):
    import torch

    import paper_2505_05950_b200 as fb
    from oracle import oracle as O2
    ref = O2.REF
    cm, _ = _ref_stack(ref, 8, E_, K_, DH, DI)
    layers, keep = _upload_stack(fb, ref, cm, 8, E_, K_, DH, DI, mixing_f16=True)
    model = fb.GpuModel(layers)
    ws = fb.Workspace(DH, DI, K_)
    hs = np.stack([O2.token_input(1, 8 * 5 + l, DH) for l in range(8)])
    y = model.decode(torch.from_numpy(hs).cuda(), ws, replay=True).cpu().numpy()
    np.save(out_path, y)


@pytest.mark.parametrize("env_var", ["FLOE_TEST_MISPREDICT", "FLOE_COOP", "FLOE_PAIRS"])
def test_launch_variants_agree(tmp_path, env_var):
    """The misprediction re-run path, the cooperative launch (no CTA pairs) and
    the unpaired launch give the default launch's outputs."""
    outs = []
    for flag in (("0", "1") if env_var != "FLOE_PAIRS" else ("1", "0")):
        out = tmp_path / f"y{flag}.npy"
        env = dict(os.environ, **{env_var: flag})
        code = (f"import sys; sys.path.insert(0, {str(ROOT)!r}); sys.path.insert(0, {str(ROOT / 'tests')!r}); "
                f"import test_gpu_multi as t; t._mispredict_run({str(out)!r})")
        r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(out))
    for l in range(8):
        assert O.rel_l2(outs[1][l], outs[0][l]) <= 1e-5, l


@pytest.mark.slow
def test_mixtral_shape_vs_per_layer_kernel(fb, torch):
    """Two of the bench's Mixtral-shaped layers (gen_model seed 7, device
    calibration): the one-launch decode equals the per-layer kernel (which
    test_gpu_parity_bench holds to the oracle at this shape)."""
    import bench
    layers, _ = bench.build_model(fb, torch, 2)
    model = fb.GpuModel(layers)
    assert model.multi_layer
    ws = fb.Workspace(bench.DH, bench.DI, bench.TOPK)
    hs = bench.replay_inputs(fb, torch, 4, 2)
    for tok in range(4):
        got = model.decode(hs[tok], ws, replay=True)
        for l in range(2):
            want = fb.layer_forward(layers[l], hs[tok][l], ws)
            assert O.rel_l2(got[l].cpu().numpy(), want.cpu().numpy()) <= 2e-2, (tok, l)
