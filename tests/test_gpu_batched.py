"""Batched up projection on the tcgen05 tensor cores (SURVEY config 4's K1):
floe_gpu_qgemv_channels_batched == qgemv_channels (quant.cpp:122-136) for every
token of the batch, within the batch-1 K1 tolerance (exact integer group sums,
f32 epilogue)."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

V_ABS, V_REL = 2e-5, 2e-5


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available()
    return torch


@pytest.fixture(scope="module")
def fb(torch):
    import paper_2505_05950_b200 as fb
    return fb


def _expert(fb, dh, di, seed):
    _, up, _ = O.seeded_expert(dh, di, seed)
    q = O.quantize(up, 2, 64)
    return q, fb.GpuExpert(dh, di, 2, 64, q.codes, q.scales, q.zeros)


def _check(q, dh, X, V, tokens):
    """|dv| <= V_ABS * rms(x_t) + V_REL * |v|: the reference's own f32 sum is
    only that accurate, and its error scales with the size of x."""
    for t in tokens:
        ref = O.qgemv_channels(q, dh, X[t])
        dv = np.abs(V[t] - ref)
        scale = float(np.sqrt(np.mean(X[t].astype(np.float64) ** 2)))
        assert np.all(dv <= V_ABS * scale + V_REL * np.abs(ref)), (t, float(dv.max()))


@pytest.fixture(scope="module")
def mixtral(fb):
    return _expert(fb, 4096, 14336, 99)


@pytest.mark.parametrize("B", [1, 5, 16, 64])
def test_batched_matches_oracle_mixtral(fb, torch, mixtral, B):
    q, e = mixtral
    X = np.stack([O.token_input(1, t, 4096) * (1.0 + 0.5 * (t % 3)) for t in range(B)])
    V = fb.qgemv_channels_batched(e, torch.from_numpy(X).cuda()).cpu().numpy()
    assert V.shape == (B, 14336)
    _check(q, 4096, X, V, range(B) if B <= 16 else [0, 1, 17, 40, B - 1])


def test_batched_agrees_with_batch1_kernel(fb, torch, mixtral):
    q, e = mixtral
    X = np.stack([O.token_input(2, t, 4096) for t in range(8)])
    V = fb.qgemv_channels_batched(e, torch.from_numpy(X).cuda()).cpu().numpy()
    ws = fb.Workspace(4096, 14336)
    for t in range(8):
        v1 = fb.qgemv_channels(e, torch.from_numpy(X[t]).cuda(), ws).cpu().numpy()
        assert np.allclose(V[t], v1, rtol=4e-5, atol=4e-5)


@pytest.mark.parametrize("dh,di,B", [(2048, 520, 7), (2048, 128, 1), (4096, 16, 33)])
def test_batched_ragged_shapes(fb, torch, dh, di, B):
    """d_intermediate not a multiple of the 128-channel block (or of a tile)."""
    q, e = _expert(fb, dh, di, 7)
    rng = np.random.default_rng(dh + di + B)
    X = rng.standard_normal((B, dh)).astype(np.float32)
    X[0] *= 1e-3  # tiny and large magnitudes in one batch
    if B > 2:
        X[2] *= 300.0
    V = fb.qgemv_channels_batched(e, torch.from_numpy(X).cuda()).cpu().numpy()
    _check(q, dh, X, V, range(B))


def test_batched_nonfinite_token_isolated(fb, torch):
    q, e = _expert(fb, 2048, 512, 3)
    X = np.stack([O.token_input(1, t, 2048) for t in range(4)])
    X[1, 100] = np.inf
    X[3, 7] = np.nan
    V = fb.qgemv_channels_batched(e, torch.from_numpy(X).cuda()).cpu().numpy()
    assert np.all(np.isnan(V[1])) and np.all(np.isnan(V[3]))
    _check(q, 2048, X, V, [0, 2])


def test_batched_argument_errors(fb, torch, mixtral):
    _, e = mixtral
    with pytest.raises(fb.FloeError):
        fb.qgemv_channels_batched(e, torch.zeros((65, 4096), device="cuda"))
    with pytest.raises(fb.FloeError):
        fb.qgemv_channels_batched(e, torch.zeros((2, 2048), device="cuda"))
    _, up, _ = O.seeded_expert(64, 256, 1)
    q = O.quantize(up, 8, 64)
    generic = fb.GpuExpert(64, 256, 8, 64, q.codes, q.scales, q.zeros)
    with pytest.raises(fb.FloeError, match="tile layout"):
        fb.qgemv_channels_batched(generic, torch.zeros((2, 64), device="cuda"))
