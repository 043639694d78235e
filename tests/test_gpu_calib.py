"""Threshold calibration on the device (floe_gpu_calib_*) against the
reference's own collect_stats + calibrate_model (model.cpp:242-330,
sparsify.cpp:42-64,128-142), compiled from its sources (oracle/_ref): the
thresholds must be BIT-IDENTICAL, on a toy multi-layer model (chained block
outputs, reservoir replacement past the cap, k in {0, 0.5, 0.8, 0.9},
drift 1 and 0.5) and on one Mixtral-shaped layer."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _float_model(L, E, dh, di, seed):
    rng = np.random.default_rng(seed)
    s = np.float32(1.0 / np.sqrt(dh))
    router = (rng.standard_normal((L, E, dh), dtype=np.float32) * s)
    mixing = (rng.standard_normal((L, dh, dh), dtype=np.float32) * s)
    gate = (rng.standard_normal((L, E, di, dh), dtype=np.float32) * s)
    up = (rng.standard_normal((L, E, di, dh), dtype=np.float32) * s)
    down = (rng.standard_normal((L, E, di, dh), dtype=np.float32) * s)
    return router, mixing, gate, up, down


def _ref_thresholds(ref, L, E, K, dh, di, w, seed, tokens, k, cap, drift):
    router, mixing, gate, up, down = (np.ascontiguousarray(a, np.float32) for a in w)
    out = np.empty(L * E, np.float32)
    rc = ref.ref_calibrate_weights(L, E, K, dh, di, router, mixing, gate, up, down, seed,
                                   tokens, k, cap, 8, drift, out)
    assert rc == 0, ref.ref_last_error()
    return out.reshape(L, E)


def _gpu_thresholds(L, E, K, dh, di, w, seed, tokens, ks, cap, drift):
    import torch

    import paper_2505_05950_b200 as fb
    router, mixing, gate, up, down = w
    cal = fb.GpuCalib(L, E, dh, di, seed, cap)
    h = torch.from_numpy(np.stack([O.token_input(seed, t, dh) for t in range(tokens)])).cuda()
    for l in range(L):
        dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
        h = cal.layer(l, dev(router[l]), dev(mixing[l]), [dev(gate[l, e]) for e in range(E)],
                      [dev(up[l, e]) for e in range(E)], [dev(down[l, e]) for e in range(E)],
                      K, h, drift_scale=drift)
    return {k: cal.thresholds(k) for k in ks}


@pytest.mark.parametrize("drift", [1.0, 0.5])
def test_calibrate_model_bit_exact_toy(ref, drift):
    L, E, K, dh, di, seed, tokens, cap = 3, 4, 2, 64, 128, 3, 10, 500
    w = _float_model(L, E, dh, di, 11)
    ks = (0.0, 0.5, 0.8, 0.9)
    got = _gpu_thresholds(L, E, K, dh, di, w, seed, tokens, ks, cap, drift)
    for k in ks:
        want = _ref_thresholds(ref, L, E, K, dh, di, w, seed, tokens, k, cap, drift)
        assert np.array_equal(got[k].view(np.uint32), want.view(np.uint32)), (k, got[k], want)


def test_calibrate_empty_expert_fails_like_reference(ref):
    import torch

    import paper_2505_05950_b200 as fb
    # one token, top-1 of 4 experts: three reservoirs stay empty
    L, E, K, dh, di = 1, 4, 1, 64, 128
    w = _float_model(L, E, dh, di, 5)
    cal = fb.GpuCalib(L, E, dh, di, 3, 500)
    h = torch.from_numpy(O.token_input(3, 0, dh)[None]).cuda()
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    cal.layer(0, dev(w[0][0]), dev(w[1][0]), [dev(w[2][0, e]) for e in range(E)],
              [dev(w[3][0, e]) for e in range(E)], [dev(w[4][0, e]) for e in range(E)], K, h)
    with pytest.raises(fb.FloeError, match="calibrate: no samples for layer 0 expert"):
        cal.thresholds(0.8)
    assert np.all(cal.thresholds(0.0) == 0.0)


@pytest.mark.slow
def test_calibrate_model_bit_exact_mixtral_layer(ref):
    """One Mixtral-shaped layer (the reference generator's streams, seed 7), 16
    calibration tokens: some reservoirs pass the 65,536 cap."""
    import torch

    import paper_2505_05950_b200 as fb
    L, E, K, dh, di, tokens = 1, 8, 2, 4096, 14336, 16
    sigma = float(np.float32(1.0) / np.sqrt(np.float32(dh)))
    base = lambda kind, e: ((0 * 5 + kind) * 65536 + e) * 64  # noqa: E731 (model.cpp:25-28)
    g = lambda kind, e, n: fb.gen_normals(7, base(kind, e), n, sigma, sharded=True)  # noqa: E731
    router, mixing = g(0, 0, E * dh).view(E, dh), g(1, 0, dh * dh).view(dh, dh)
    gate = [g(2, e, dh * di).view(di, dh) for e in range(E)]
    up = [g(3, e, dh * di).view(di, dh) for e in range(E)]
    down = [g(4, e, dh * di).view(di, dh) for e in range(E)]
    cal = fb.GpuCalib(L, E, dh, di, 3)
    h = torch.from_numpy(np.stack([O.token_input(3, t, dh) for t in range(tokens)])).cuda()
    cal.layer(0, router, mixing, gate, up, down, K, h, want_next=False)
    got = cal.thresholds(0.8)
    host = lambda ts: np.stack([t.cpu().numpy() for t in ts])[None]  # noqa: E731
    w = (router.cpu().numpy()[None], mixing.cpu().numpy()[None], host(gate), host(up), host(down))
    want = _ref_thresholds(ref, L, E, K, dh, di, w, 3, tokens, 0.8, 1 << 16, 1.0)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (got, want)
