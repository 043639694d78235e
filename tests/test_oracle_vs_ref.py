"""The C restatement against the live reference library, on random cases.

Needs oracle/_ref/libfloe_ref.so (built from /root/reference by oracle/Makefile;
the prebuilt .so also travels to the GPU box).  Bit-exact throughout.
"""
import ctypes as ct

import numpy as np
import pytest

from oracle import oracle as O


def beq(a, b):
    return np.array_equal(np.asarray(a).view(np.uint8), np.asarray(b).view(np.uint8))


@pytest.mark.parametrize("seed,stream,n", [(0, 0, 1), (7, 3, 777), (2**40, 5, 10001)])
def test_normals(ref, seed, stream, n):
    b = np.empty(n, np.float32)
    ref.ref_normals(seed, stream, n, b)
    assert beq(O.normals(seed, stream, n), b)


def test_f32_to_f16_random_bits(ref):
    x = np.frombuffer(np.random.default_rng(3).bytes(4 << 18), np.float32).copy()
    x = x[np.isfinite(x)]
    h = np.empty(x.size, np.uint16)
    ref.ref_f32_to_f16(x, x.size, h)
    assert beq(O.f32_to_f16(x), h)


@pytest.mark.parametrize("bits", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("g", [8, 64])
def test_quantize_qgemv_dequantize(ref, bits, g):
    dh, di = 64, 40
    x = O.normals(5, 1, dh * di, 0.125)
    q = O.quantize(x, bits, g)
    c2, s2, z2 = np.zeros_like(q.codes), np.zeros_like(q.scales), np.zeros_like(q.zeros)
    assert ref.ref_quantize(x, x.size, bits, g, c2, s2, z2) == 0
    assert beq(q.codes, c2) and beq(q.scales, s2) and beq(q.zeros, z2)
    xin = O.normals(6, 2, dh)
    v2 = np.empty(di, np.float32)
    assert ref.ref_qgemv_channels(q.codes, q.scales, q.zeros, q.n, bits, g, dh, xin, v2) == 0
    assert beq(O.qgemv_channels(q, dh, xin), v2)
    d2 = np.empty(q.n, np.float32)
    assert ref.ref_dequantize(q.codes, q.scales, q.zeros, q.n, bits, g, d2) == 0
    assert beq(O.dequantize(q), d2)


def test_quantize_errors_match(ref):
    x = O.normals(1, 1, 16)
    for bits, g in [(5, 8), (2, 5)]:
        with pytest.raises(ValueError) as ei:
            O.quantize(x, bits, g)
        c = np.zeros(16, np.uint8)
        s = np.zeros(16, np.uint16)
        assert ref.ref_quantize(x, 16, bits, g, c, s, s.copy()) != 0
        assert O.ref_error() == str(ei.value)
    bad = x.copy()
    bad[3] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        O.quantize(bad, 2, 8)


@pytest.mark.parametrize("k", [0.0, 0.5, 0.8, 0.9, 1.0])
def test_expert_forward_sparse(ref, k):
    dh, di = 128, 192
    gate, up, down = O.seeded_expert(dh, di, 77)
    x = O.seeded_input(dh, 78)
    q = O.quantize(up, 2, 64)
    v = O.qgemv_channels(q, dh, x)
    t = O.calibrate_threshold(np.abs(v), k)
    assert np.float32(t) == np.float32(ref.ref_calibrate_threshold(np.abs(v), di, k))
    e = O.Expert(dh, di, q, gate, down, t)
    h = ref.ref_expert_create(dh, di, 2, 64, q.codes, q.scales, q.zeros, gate, down, t)
    y2 = np.empty(dh, np.float32)
    assert ref.ref_expert_forward(h, x, y2) == 0
    ref.ref_expert_destroy(h)
    assert beq(O.expert_forward_sparse(e, x), y2)


def test_dense_expert(ref):
    dh, di = 32, 48
    gate, up, down = O.seeded_expert(dh, di, 5)
    x = O.seeded_input(dh, 6)
    y2 = np.empty(dh, np.float32)
    assert ref.ref_expert_forward_dense(dh, di, gate, up, down, x, y2) == 0
    assert beq(O.expert_forward_dense(dh, di, gate, up, down, x), y2)


def test_route_topk_ties(ref):
    for trial in range(50):
        rng = np.random.default_rng(trial)
        E, dh, k = 8, 16, int(rng.integers(1, 9))
        router = rng.integers(-2, 3, size=(E, dh)).astype(np.float32)  # many exact ties
        u = rng.integers(-2, 3, size=dh).astype(np.float32)
        s2 = np.empty(k, np.uint32)
        w2 = np.empty(k, np.float32)
        assert ref.ref_route(router, E, dh, u, k, s2, w2) == 0
        s1, w1 = O.route(router, u, k)
        assert np.array_equal(s1, s2) and beq(w1, w2)


def test_predict_mask_and_experts(ref):
    dh, di = 64, 96
    _, up, _ = O.seeded_expert(dh, di, 9)
    q = O.quantize(up, 2, 32)
    xp = O.seeded_input(dh, 10)
    m2 = np.empty(di, np.uint8)
    assert ref.ref_predict_mask(q.codes, q.scales, q.zeros, q.n, 2, 32, dh, xp, 0.7, m2) == 0
    assert np.array_equal(O.predict_mask(q, dh, xp, 0.7), m2)
    W = O.normals(3, 3, 8 * dh).reshape(8, dh)
    b = O.normals(3, 4, 8)
    o2 = np.empty(3, np.uint32)
    assert ref.ref_predict_experts(W, b, 8, dh, xp, 3, o2) == 0
    assert np.array_equal(O.predict_experts(W, b, xp, 3), o2)


@pytest.mark.parametrize("eb", [2, 4])
def test_pack_compact(ref, eb):
    dh, di = 32, 40
    gate, up, down = O.seeded_expert(dh, di, 12)
    q = O.quantize(up, 2, 32)
    e = O.Expert(dh, di, q, gate, down, 0.0)
    mask = (np.arange(di) % 3 == 0).astype(np.uint8)
    ch1, p1 = O.pack_compact(e, mask, eb)
    h = ref.ref_expert_create(dh, di, 2, 32, q.codes, q.scales, q.zeros, gate, down, 0.0)
    ch2 = np.empty(di, np.uint32)
    p2 = np.empty(di * 2 * dh * eb, np.uint8)
    n = ct.c_uint64()
    assert ref.ref_pack_compact(h, mask, eb, ch2, p2, ct.byref(n)) == 0
    ref.ref_expert_destroy(h)
    assert np.array_equal(ch1, ch2[: n.value]) and beq(p1, p2[: n.value * 2 * dh * eb])


@pytest.mark.slow
def test_mixtral_qgemv_prefix(ref):
    """Config-1 weights: the parallel skip-ahead generator and the group-fast
    qgemv equal the reference on the first 64 channels at Mixtral shape."""
    dh, di = 4096, 14336
    gate, up, down = O.seeded_expert(dh, di, 99)
    n = 64 * dh
    b = np.empty(n, np.float32)
    ref.ref_normals(99, 2, n, b)
    sd = np.float32(1.0) / np.sqrt(np.float32(dh))
    assert beq(b * sd, up[:n])
    q = O.quantize(up[:n], 2, 64)
    x = O.seeded_input(dh, 100)
    v2 = np.empty(64, np.float32)
    assert ref.ref_qgemv_channels(q.codes, q.scales, q.zeros, n, 2, 64, dh, x, v2) == 0
    assert beq(O.qgemv_channels(q, dh, x), v2)
