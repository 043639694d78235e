"""Pin the C restatement (oracle/floe_oracle.c) to the reference's own outputs.

The fixtures in tests/golden/ were produced by tests/golden/make_golden.py from
the UNMODIFIED reference core (oracle/_ref/libfloe_ref.so).  These tests need
no reference at run time, so they also pin the oracle on the GPU box.
Everything here is bit-exact: integer, byte and IEEE-f32 outputs of the same
operation order.
"""
import numpy as np
import pytest

from oracle import oracle as O

EXPERTS = ["expert_acc1_b8", "expert_b2_g64", "expert_b4_g32", "expert_b3_g8",
           "expert_b2_dh2048"]


def bits_equal(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8))


def test_f16_conversions(golden):
    g = golden("scalars")
    assert bits_equal(O.f32_to_f16(g["f32_in"]), g["f16_out"])
    assert bits_equal(O.f16_to_f32(np.arange(65536, dtype=np.uint16)), g["f16_all"])


def test_rng_streams(golden):
    g = golden("scalars")
    assert bits_equal(O.normals(99, 1, 1001), g["normals_99_1"])
    assert bits_equal(O.token_input(1, 5, 64), g["token_1_5"])


def test_topk_softmax_ratio(golden):
    g = golden("scalars")
    assert np.array_equal(O.top_k(g["topk_in"], 3), g["topk_out"])
    sm = np.array([1.0, 2.0, 3.0], np.float32)
    O.C.fo_softmax_inplace(sm, 3)
    assert bits_equal(sm, g["softmax_out"])
    r = [O.C.fo_compression_ratio(4096, 14336, 2, 64, 0.10, 0),
         O.C.fo_compression_ratio(4096, 14336, 2, 64, 0.10, 1)]
    assert r == list(g["ratios"])


@pytest.mark.parametrize("name", EXPERTS)
def test_expert_fixture(golden, name):
    g = golden(name)
    dh, di, bits, gs = int(g["dh"]), int(g["di"]), int(g["bits"]), int(g["group_size"])
    gate, up, down = O.seeded_expert(dh, di, int(g["seed"]))
    assert bits_equal(gate, g["gate"]) and bits_equal(up, g["up"]) and bits_equal(down, g["down"])
    x = O.seeded_input(dh, int(g["xseed"]))
    assert bits_equal(x, g["x"])
    q = O.quantize(up, bits, gs)
    assert bits_equal(q.codes, g["codes"])
    assert bits_equal(q.scales, g["scales"]) and bits_equal(q.zeros, g["zeros"])
    assert bits_equal(O.dequantize(q), g["deq"])
    v = O.qgemv_channels(q, dh, x)
    assert bits_equal(v, g["v"])
    t = O.calibrate_threshold(np.abs(v), float(g["k"]))
    assert np.float32(t) == g["threshold"]
    e = O.Expert(dh, di, q, gate, down, t)
    y, v2, mask = O.expert_forward_sparse(e, x, want_v=True)
    assert bits_equal(y, g["y"])
    assert bits_equal(mask, g["mask"])
    e16 = O.Expert(dh, di, q, O.fp16_round(gate), O.fp16_round(down), t)
    assert bits_equal(O.expert_forward_sparse(e16, x), g["y_f16"])
    ch, payload = O.pack_compact(e, mask, 2)
    assert np.array_equal(ch, g["pack_channels"])
    assert bits_equal(payload, g["pack_payload"])


def toy_layer(g, l):
    E, K, dh, di = int(g["E"]), int(g["K"]), int(g["dh"]), int(g["di"])
    experts = []
    for e in range(E):
        q = O.Quantized(g[f"codes{l}_{e}"], g[f"scales{l}_{e}"], g[f"zeros{l}_{e}"], dh * di,
                        int(g["bits"]), int(g["group_size"]))
        experts.append(O.Expert(dh, di, q, g[f"gate{l}_{e}"], g[f"down{l}_{e}"],
                                float(g[f"threshold{l}_{e}"])))
    return O.Layer(g[f"router{l}"].reshape(E, dh), g[f"mixing{l}"].reshape(dh, dh), experts, K)


def test_toy_layer_traced(golden):
    g = golden("toy_layer")
    L = int(g["L"])
    layers = [toy_layer(g, l) for l in range(L)]
    for i in range(int(g["n_steps"])):
        tr = O.layer_forward(layers[i % L], g[f"tok{i}_h"], traced=True)
        assert bits_equal(tr["block_input"], g[f"tok{i}_u"])
        assert np.array_equal(tr["experts"], g[f"tok{i}_sel"])
        assert bits_equal(tr["weights"], g[f"tok{i}_w"])
        assert np.array_equal(tr["masks"], g[f"tok{i}_masks"])
        assert bits_equal(tr["out"], g[f"tok{i}_y"])
