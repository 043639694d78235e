"""The prefill expert forward (floe_gpu_expert_forward_prefill): dense f16
tensor-core GEMMs with hi/lo splits for many tokens per expert (config 5).
Per token it must be expert_forward_sparse (model.cpp:128-142): equal to the
single-token fused kernel (same masks up to ties) and to the reference within
1e-2, at any token magnitude (per-token power-of-two scales)."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


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
def mixtral(fb):
    dh, di = 4096, 14336
    gate, up, down = O.seeded_expert(dh, di, 99)
    q = O.quantize(up, 2, 64)
    x0 = O.seeded_input(dh, 100)
    t = O.calibrate_threshold(np.abs(O.qgemv_channels(q, dh, x0)), 0.8)
    e = fb.GpuExpert(dh, di, 2, 64, q.codes, q.scales, q.zeros, gate=gate, down=down, threshold=t)
    return O.Expert(dh, di, q, gate, down, t), e


@pytest.mark.parametrize("n", [1, 37, 300])
def test_prefill_matches_single_token_and_reference(fb, torch, mixtral, n):
    ref_e, e = mixtral
    X = np.stack([O.seeded_input(4096, 500 + t) for t in range(n)])
    if n > 2:
        X[1] *= 300.0   # coefficients ~1e5: past f16's range without the row scale
        X[2] *= 1e-3    # keeps nothing at this threshold: y = 0
    xd = torch.from_numpy(X).cuda()
    Y = fb.expert_forward_prefill(e, xd).cpu().numpy()
    ws = fb.Workspace(4096, 14336)
    for t in sorted({0, 1, 2, n - 1} & set(range(n))):
        y1 = fb.expert_forward_sparse(e, xd[t], ws).cpu().numpy()
        if np.linalg.norm(y1) == 0:
            assert np.linalg.norm(Y[t]) == 0, t
            continue
        # same arithmetic up to summation order; a channel at |v| ~ t may flip
        assert O.rel_l2(Y[t], y1) <= 2e-3, (t, O.rel_l2(Y[t], y1))
    for t in (0, n - 1):
        assert O.rel_l2(Y[t], O.expert_forward_sparse(ref_e, X[t])) <= 1e-2, t


def test_prefill_small_scale_tokens(fb, torch, mixtral):
    """Tokens x1e-3 against a threshold scaled the same way (every product in
    f16's subnormal range without the per-row scales)."""
    ref_e, _ = mixtral
    q = ref_e.up_q
    small = fb.GpuExpert(4096, 14336, 2, 64, q.codes, q.scales, q.zeros, gate=ref_e.gate,
                         down=ref_e.down_t, threshold=ref_e.threshold * 1e-3)
    X = np.stack([O.seeded_input(4096, 700 + t) for t in range(20)]) * 1e-3
    xd = torch.from_numpy(X.astype(np.float32)).cuda()
    Y = fb.expert_forward_prefill(small, xd).cpu().numpy()
    ws = fb.Workspace(4096, 14336)
    for t in (0, 7, 19):
        y1 = fb.expert_forward_sparse(small, xd[t], ws).cpu().numpy()
        assert np.linalg.norm(y1) > 0
        assert O.rel_l2(Y[t], y1) <= 2e-3, t


def test_prefill_nonfinite_token_isolated(fb, torch, mixtral):
    _, e = mixtral
    X = np.stack([O.seeded_input(4096, 800 + t) for t in range(4)])
    X[1, 5] = np.nan
    Y = fb.expert_forward_prefill(e, torch.from_numpy(X).cuda()).cpu().numpy()
    assert np.all(np.isnan(Y[1]))
    assert np.all(np.isfinite(Y[[0, 2, 3]]))
