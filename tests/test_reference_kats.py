"""Known-answer tests of the reference suites, re-hosted on the C oracle.

The reference's doctest binaries cannot build here (vendor/doctest.h is absent,
SURVEY.md §4), so the hot-path cases are restated against oracle/liboracle.so,
each citing the reference test it re-hosts (proj/tests/...).
"""
import numpy as np
import pytest

from oracle import oracle as O


def gaussian_vec(n, seed):  # test_quant.cpp:15-20 (Rng(seed), stream 0)
    return O.normals(seed, 0, n)


def test_constant_roundtrip():  # test_quant.cpp:47-52
    q = O.quantize(np.full(32, 0.375, np.float32), 2, 8)
    assert np.all(O.dequantize(q) == 0.375)


def test_integer_ramp_bits2():  # test_quant.cpp:54-62
    q = O.quantize(np.array([0, 1, 2, 3], np.float32), 2, 4)
    assert O.f16_to_f32(q.scales)[0] == 1.0 and O.f16_to_f32(q.zeros)[0] == 0.0
    assert np.array_equal(O.dequantize(q), np.array([0, 1, 2, 3], np.float32))
    assert q.codes[0] == 0b11100100


def test_all_zero():  # test_quant.cpp:64-70
    q = O.quantize(np.zeros(64, np.float32), 4, 16)
    assert np.all(q.codes == 0) and np.all(O.dequantize(q) == 0)


@pytest.mark.parametrize("bits", [2, 8])
def test_roundtrip_half_scale(bits):  # test_quant.cpp:72-82
    v = gaussian_vec(64 * 64, 7)
    q = O.quantize(v, bits, 64)
    back = O.dequantize(q)
    scale = np.repeat(O.f16_to_f32(q.scales), 64)
    assert np.all(np.abs(v - back) <= scale / 2 + 1e-6)


def test_requantize_fixed_point():  # test_quant.cpp:103-112
    v = gaussian_vec(256, 9)
    for bits in (1, 2, 3, 4, 8):
        q = O.quantize(v, bits, 32)
        q2 = O.quantize(O.dequantize(q), bits, 32)
        assert np.array_equal(q.codes, q2.codes)
        assert np.array_equal(q.scales, q2.scales) and np.array_equal(q.zeros, q2.zeros)


def test_byte_straddle_packing():  # test_quant.cpp:114-121 (independent bit reader)
    v = gaussian_vec(16, 10)
    for bits in (1, 2, 3, 4, 8):
        q = O.quantize(v, bits, 8)
        allbits = np.unpackbits(q.codes, bitorder="little")
        codes = [int(sum(int(allbits[i * bits + b]) << b for b in range(bits))) for i in range(16)]
        # dequantize must see the same codes as the bitwise reader
        deq = O.dequantize(q)
        sc = np.repeat(O.f16_to_f32(q.scales), 8)
        ze = np.repeat(O.f16_to_f32(q.zeros), 8)
        assert np.array_equal(deq, np.array(codes, np.float32) * sc + ze)


def test_mse_monotone_in_bits():  # test_quant.cpp:123-131
    v = gaussian_vec(1024, 11)
    prev = 1e30
    for bits in (1, 2, 3, 4, 8):
        e = float(np.mean((v.astype(np.float64) - O.dequantize(O.quantize(v, bits, 64))) ** 2))
        assert e <= prev + 1e-12
        prev = e


def test_invalid_args():  # test_quant.cpp:133-140
    v = gaussian_vec(16, 12)
    with pytest.raises(ValueError):
        O.quantize(v, 5, 8)
    with pytest.raises(ValueError):
        O.quantize(v, 2, 5)


def test_production_bytes():  # test_quant.cpp:142-153
    n = 4096 * 14336
    assert O.C.fo_packed_code_bytes(n, 2) == 14680064
    assert 14680064 + 4 * (n // 64) == 14680064 + 4 * 917504


def test_qgemv_equals_dequant_gemv():  # test_quant.cpp:162-177
    ch, ln = 8, 16
    q = O.quantize(gaussian_vec(ch * ln, 14), 4, 16)
    x = gaussian_vec(ln, 15)
    deq = O.dequantize(q).reshape(ch, ln)
    ref = np.empty(ch, np.float32)
    O.C.fo_gemv(ch, ln, np.ascontiguousarray(deq), x, ref)
    assert np.array_equal(O.qgemv_channels(q, ln, x).view(np.uint32), ref.view(np.uint32))


def test_compression_ratio():  # test_quant.cpp:179-186 / acceptance check 4
    nominal = O.C.fo_compression_ratio(4096, 14336, 2, 64, 0.10, 0)
    meta = O.C.fo_compression_ratio(4096, 14336, 2, 64, 0.10, 1)
    assert 9.0 <= nominal <= 9.5 and meta >= 8.0 and meta < nominal
    assert f"{nominal:.4f}" == "9.2292" and f"{meta:.4f}" == "8.4197"


def masked_dense(e, x, v, t):  # acceptance_test.cpp:86-97
    dh, di = e.d_hidden, e.d_intermediate
    y = np.zeros(dh, np.float32)
    g = e.gate.reshape(di, dh)
    d = e.down_t.reshape(di, dh)
    for c in range(di):
        s = np.float32(O.C.fo_silu(np.float32(np.dot(g[c], x)))) * v[c] if abs(v[c]) >= t \
            else np.float32(0)
        y += np.float32(s) * d[c]
    return y


def test_acceptance_check1_sample():  # acceptance_test.cpp:107-141 (20 of 1000 trials)
    for trial in range(20):
        gate, up, down = O.seeded_expert(64, 256, 1000 + trial)
        x = O.seeded_input(64, 2000 + trial)
        e = O.compress_expert(64, 256, gate, up, down, 8, 64, 0.0)
        v = O.qgemv_channels(e.up_q, 64, x)
        e.threshold = O.calibrate_threshold(np.abs(v), 0.5)
        got = O.expert_forward_sparse(e, x)
        assert O.rel_l2(got, masked_dense(e, x, v, e.threshold)) <= 1e-5
        e.threshold = 0.0
        got0 = O.expert_forward_sparse(e, x)
        dense = O.expert_forward_dense(64, 256, gate, O.dequantize(e.up_q), down, x)
        assert O.rel_l2(got0, dense) <= 1e-3


def test_acceptance_check2_nan_poison():  # acceptance_test.cpp:145-176 (100 trials)
    for trial in range(100):
        gate, up, down = O.seeded_expert(16, 32, 5000 + trial)
        x = O.seeded_input(16, 6000 + trial)
        e = O.compress_expert(16, 32, gate, up, down, 8, 16, 0.0)
        v = O.qgemv_channels(e.up_q, 16, x)
        e.threshold = O.calibrate_threshold(np.abs(v), 0.5)
        clean = O.expert_forward_sparse(e, x)
        pg, pd = e.gate.reshape(32, 16).copy(), e.down_t.reshape(32, 16).copy()
        drop = np.abs(v) < e.threshold
        pg[drop] = np.nan
        pd[drop] = np.nan
        pe = O.Expert(16, 32, e.up_q, pg, pd, e.threshold)
        got = O.expert_forward_sparse(pe, x)
        assert np.all(np.isfinite(got)) and np.array_equal(got, clean)


def test_threshold_above_max_gives_zero():  # test_model.cpp:129-134
    gate, up, down = O.seeded_expert(8, 16, 6)
    e = O.compress_expert(8, 16, gate, up, down, 8, 8, 1e6)
    assert np.all(O.expert_forward_sparse(e, O.seeded_input(8, 7, 9)) == 0)


def test_keep_on_equality():  # test_sparsify.cpp:46-50
    v = np.array([0.5, -0.5, 0.49999997, 1.0], np.float32)
    assert list(O.sparsity_mask(v, 0.5)) == [1, 1, 0, 1]
    assert list(O.sparsity_mask(v, 0.0)) == [1, 1, 1, 1]


def test_routing_kats():  # test_model.cpp:150-169
    sel, w = O.route(np.zeros((2, 4), np.float32), O.seeded_input(4, 10, 9), 2)
    assert list(sel) == [0, 1] and list(w) == [0.5, 0.5]
    r = O.normals(11, 0, 12).reshape(3, 4)
    sel, w = O.route(r, O.seeded_input(4, 12, 9), 1)
    assert len(sel) == 1 and w[0] == 1.0


def test_compact_record_bytes():  # test_offload.cpp:79-89
    assert O.C.fo_channel_record_bytes(4096, 2) == 16384


def test_reuse_mask_zero_drift():  # test_predictor.cpp:188-209 (x_prev == x: exact)
    dh, di = 32, 64
    _, up, _ = O.seeded_expert(dh, di, 3)
    q = O.quantize(up, 8, 32)
    x = O.seeded_input(dh, 4)
    v = O.qgemv_channels(q, dh, x)
    t = O.calibrate_threshold(np.abs(v), 0.5)
    assert np.array_equal(O.predict_mask(q, dh, x, t), (np.abs(v) >= t).astype(np.uint8))
    assert np.all(O.predict_mask(q, dh, x, 0.0) == 1)
