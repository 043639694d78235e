"""Batched up projection on the tcgen05 tensor cores (SURVEY config 4's K1):
floe_gpu_qgemv_channels_batched == qgemv_channels (quant.cpp:122-136) for every
token of the batch, within the batch-1 K1 tolerance (exact integer group sums,
f32 epilogue)."""
import numpy as np
from pathlib import Path
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


@pytest.mark.parametrize("dh,di,B", [(2048, 520, 7), (2048, 128, 1), (4096, 16, 33), (4096, 24, 5),
                                     (2048, 40, 16)])
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


@pytest.mark.parametrize("B", [9, 12])
def test_small_batch_imma_path_two_passes(fb, torch, mixtral, B):
    """<= 16 tokens run on the IMMA kernel (floe_k1b.cuh) in passes of 8: a
    partial second pass, every token against the oracle."""
    q, e = mixtral
    X = np.stack([O.token_input(4, t, 4096) * (1.0 + 0.25 * t) for t in range(B)])
    V = fb.qgemv_channels_batched(e, torch.from_numpy(X).cuda()).cpu().numpy()
    _check(q, 4096, X, V, range(B))


def test_imma_and_tcgen05_paths_agree(fb, torch, mixtral):
    """16 tokens take the IMMA kernel, 17 the tcgen05 kernel: the same exact
    integer span sums and per-span f32 steps, so the shared tokens agree to the
    last few ulps (only the order of the final partial sums differs)."""
    _, e = mixtral
    X = np.stack([O.token_input(5, t, 4096) for t in range(17)])
    Xd = torch.from_numpy(X).cuda()
    V16 = fb.qgemv_channels_batched(e, Xd[:16]).cpu().numpy()
    V17 = fb.qgemv_channels_batched(e, Xd).cpu().numpy()
    scale = np.abs(V17[:16]).max()
    assert np.max(np.abs(V16 - V17[:16])) <= 1e-6 * scale


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


# ------------------------------------------------ batched expert forward
@pytest.fixture(scope="module")
def mixtral_full(fb):
    dh, di = 4096, 14336
    gate, up, down = O.seeded_expert(dh, di, 99)
    q = O.quantize(up, 2, 64)
    x0 = O.seeded_input(dh, 100)
    t = O.calibrate_threshold(np.abs(O.qgemv_channels(q, dh, x0)), 0.8)
    e = fb.GpuExpert(dh, di, 2, 64, q.codes, q.scales, q.zeros, gate=gate, down=down, threshold=t)
    return O.Expert(dh, di, q, gate, down, t), e


@pytest.mark.parametrize("B", [1, 3, 4, 7, 16, 64])
def test_expert_forward_batched_matches_per_token(fb, torch, mixtral_full, B):
    """Each token of the batch == the single-token fused path on the same
    token (same masks up to exact ties), and == the reference within 1e-2."""
    ref_e, e = mixtral_full
    X = np.stack([O.seeded_input(4096, 100 + t) for t in range(B)])
    xd = torch.from_numpy(X).cuda()
    v = torch.empty((B, 14336), dtype=torch.float32, device="cuda")
    Y = fb.expert_forward_batched(e, xd, v=v).cpu().numpy()
    ws = fb.Workspace(4096, 14336)
    for t in (range(B) if B <= 16 else [0, 5, 31, 63]):
        y1 = fb.expert_forward_sparse(e, xd[t], ws).cpu().numpy()
        assert O.rel_l2(Y[t], y1) <= 1e-4, t
        if t < 3:
            assert O.rel_l2(Y[t], O.expert_forward_sparse(ref_e, X[t])) <= 1e-2
    V = v.cpu().numpy()
    _check(ref_e.up_q, 4096, X, V, [0, B - 1])


@pytest.mark.parametrize("B", [16, 33])
def test_expert_forward_batched_token_scales(fb, torch, mixtral_full, B):
    """The tcgen05 gate/down GEMMs split x and the coefficients into f16 hi+lo
    with a per-token power-of-two scale: tokens x300 (coefficients ~1e5, past
    f16's range unscaled) and x1e-3 (against a threshold scaled the same way,
    coefficients in f16's subnormals unscaled) equal the single-token path."""
    ref_e, e = mixtral_full
    q = ref_e.up_q
    X = np.stack([O.seeded_input(4096, 300 + t) for t in range(B)])
    X[1] *= 300.0
    X[4] *= 300.0
    ws = fb.Workspace(4096, 14336)
    Y = fb.expert_forward_batched(e, torch.from_numpy(X).cuda()).cpu().numpy()
    for t in (0, 1, 4, B - 1):
        y1 = fb.expert_forward_sparse(e, torch.from_numpy(X[t]).cuda(), ws).cpu().numpy()
        assert O.rel_l2(Y[t], y1) <= 1e-4, t
    small = fb.GpuExpert(4096, 14336, 2, 64, q.codes, q.scales, q.zeros, gate=ref_e.gate,
                         down=ref_e.down_t, threshold=ref_e.threshold * 1e-3)
    Xs = X * 1e-3
    Xs[1] = X[1] / 300.0 * 1e-3
    Xs[4] = X[4] / 300.0 * 1e-3
    Ys = fb.expert_forward_batched(small, torch.from_numpy(Xs).cuda()).cpu().numpy()
    for t in (0, 2, B - 1):
        y1 = fb.expert_forward_sparse(small, torch.from_numpy(Xs[t]).cuda(), ws).cpu().numpy()
        assert np.linalg.norm(y1) > 0, t
        assert O.rel_l2(Ys[t], y1) <= 1e-4, t


def test_expert_forward_batched_small_and_edge(fb, torch):
    """Ragged shape, a threshold that keeps nothing for some tokens, and a
    token with a non-finite input (its NaN v keeps every channel, as the
    reference's `fabs(v) < t` test does) next to finite ones."""
    dh, di = 2048, 520
    gate, up, down = O.seeded_expert(dh, di, 11)
    q = O.quantize(up, 2, 64)
    X = np.stack([O.token_input(1, t, dh) * (0.05 if t == 1 else 1.0) for t in range(5)])
    t_hi = O.calibrate_threshold(np.abs(O.qgemv_channels(q, dh, X[0])), 0.9)
    e = fb.GpuExpert(dh, di, 2, 64, q.codes, q.scales, q.zeros, gate=gate, down=down,
                     threshold=t_hi)
    ref_e = O.Expert(dh, di, q, gate, down, t_hi)
    X[3, 9] = np.nan
    Y = fb.expert_forward_batched(e, torch.from_numpy(X).cuda()).cpu().numpy()
    ws = fb.Workspace(dh, di)
    for t in (0, 1, 2, 4):
        y1 = fb.expert_forward_sparse(e, torch.from_numpy(X[t]).cuda(), ws).cpu().numpy()
        if np.linalg.norm(y1) == 0:
            assert np.all(Y[t] == 0)
        else:
            assert O.rel_l2(Y[t], y1) <= 1e-4
        assert O.rel_l2(Y[t], O.expert_forward_sparse(ref_e, X[t])) <= 1e-2 or np.linalg.norm(y1) == 0
    assert np.all(np.isnan(Y[3]))


def test_gate_gemm_and_cuda_core_paths_agree(tmp_path):
    """The gate dots and the down product of the batched forward run as tcgen05
    f16 GEMMs (x / the coefficients split into hi + lo halves) or on CUDA
    cores; all four combinations give the same outputs."""
    import os
    import subprocess
    import sys
    root = __import__("pathlib").Path(__file__).resolve().parents[1]
    code = (
        "import sys, numpy as np, torch; sys.path.insert(0, %r)\n"
        "from oracle import oracle as O\n"
        "import paper_2505_05950_b200 as fb\n"
        "gate, up, down = O.seeded_expert(2048, 1040, 21)\n"
        "q = O.quantize(up, 2, 64)\n"
        "e = fb.GpuExpert(2048, 1040, 2, 64, q.codes, q.scales, q.zeros, gate=gate, down=down, threshold=1.0)\n"
        "X = torch.from_numpy(np.stack([O.token_input(4, t, 2048) for t in range(24)])).cuda()\n"
        "np.save(sys.argv[1], fb.expert_forward_batched(e, X).cpu().numpy())\n") % str(root)
    outs = []
    for gate, down in (("0", "0"), ("1", "0"), ("0", "1"), ("1", "1")):
        f = tmp_path / f"y{gate}{down}.npy"
        r = subprocess.run([sys.executable, "-c", code, str(f)], cwd=root, capture_output=True,
                           text=True, timeout=300,
                           env=dict(os.environ, FLOE_GATE_TC=gate, FLOE_DOWN_TC=down))
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(f))
    for o in outs[1:]:
        for t in range(24):
            assert O.rel_l2(o[t], outs[0][t]) <= 1e-5, t


def _union_paths_run(out_path):
    import torch

    import paper_2505_05950_b200 as fb2
    from oracle import oracle as O2
    gate, up, down = O2.seeded_expert(2048, 1000, 21)
    q = O2.quantize(up, 2, 64)
    t = O2.calibrate_threshold(np.abs(O2.qgemv_channels(q, 2048, O2.seeded_input(2048, 1))), 0.8)
    e = fb2.GpuExpert(2048, 1000, 2, 64, q.codes, q.scales, q.zeros, gate=gate, down=down, threshold=t)
    X = torch.from_numpy(np.stack([O2.token_input(1, 40 + i, 2048) for i in range(7)])).cuda()
    outs = [fb2.expert_forward_batched(e, X[:b]).cpu().numpy() for b in (1, 2, 4, 7)]
    np.savez(out_path, *outs)


def test_fused_union_kernel_matches_two_kernel_path(tmp_path):
    """<= 8 tokens: the fused union gate/down kernel (union_ffn, groups of <= 4
    tokens) == the coeffs + down_accum path (FLOE_UNION_FUSED=0) up to
    summation order."""
    import os
    import subprocess
    import sys
    res = {}
    for flag in ("1", "0"):
        out = tmp_path / f"u{flag}.npz"
        code = (f"import sys; sys.path.insert(0, {str(Path(__file__).resolve().parents[1])!r}); "
                f"sys.path.insert(0, {str(Path(__file__).resolve().parent)!r}); "
                f"import test_gpu_batched as T; T._union_paths_run({str(out)!r})")
        env = dict(os.environ, FLOE_UNION_FUSED=flag)
        subprocess.run([sys.executable, "-c", code], check=True, env=env, timeout=600)
        res[flag] = np.load(out)
    for k in res["1"].files:
        a, b = res["1"][k], res["0"][k]
        assert O.rel_l2(a, b) <= 1e-5, k

