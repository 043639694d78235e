"""FLOR record-cache files: the device image of a
compressed model with f16 gate|down records, the device-friendly counterpart
of FLOQ (load_compressed, core/src/model.cpp:414-474).  A saved and reloaded
stack routes and masks bit-identically; the up projection round-trips to the
reference packing bit-exactly (expert_download inverts the tile layout)."""
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


@pytest.mark.parametrize("dh,di,bits,g", [(4096, 1024, 2, 64), (2048, 512, 2, 128), (64, 256, 8, 64)])
def test_expert_download_round_trips_reference_packing(fb, dh, di, bits, g):
    _, up, _ = O.seeded_expert(dh, di, 21)
    q = O.quantize(up, bits, g)
    e = fb.GpuExpert(dh, di, bits, g, q.codes, q.scales, q.zeros, threshold=0.75)
    d = e.download()
    assert np.array_equal(d["codes"], q.codes)
    assert np.array_equal(d["scales"], q.scales) and np.array_equal(d["zeros"], q.zeros)
    assert d["threshold"] == np.float32(0.75)


@pytest.mark.parametrize("mixing_f16,host", [(True, False), (False, True)])
def test_record_cache_round_trip(fb, torch, tmp_path, mixing_f16, host):
    L, E, K, dh, di = 2, 4, 2, 2048, 512
    rng = np.random.default_rng(4)
    layers = []
    for l in range(L):
        ex = []
        for e in range(E):
            gate, up, down = O.seeded_expert(dh, di, 60 * l + e)
            q = O.quantize(up, 2, 64)
            ex.append(fb.GpuExpert(dh, di, 2, 64, q.codes, q.scales, q.zeros, gate=gate, down=down,
                                   threshold=0.9 + 0.01 * e))
        router = (rng.standard_normal((E, dh)) / 45).astype(np.float32)
        mixing = (rng.standard_normal((dh, dh)) / 45).astype(np.float32)
        layers.append(fb.GpuLayer(router, mixing, ex, K, mixing_f16=mixing_f16))
    path = tmp_path / "m.flor"
    fb.save_record_cache(path, layers)
    info = fb.record_cache_info(path)
    n = dh * di
    per_expert = 64 + n * 2 // 8 + 2 * (2 * n // 64) + 4 * n  # all sections 64-B multiples here
    per_layer = 4 * E * dh + dh * dh * (2 if mixing_f16 else 4) + E * per_expert
    assert info["file_bytes"] == 64 + L * per_layer
    assert (info["layers"], info["experts"], info["top_k"], info["d_hidden"]) == (L, E, K, dh)
    assert info["mixing_f16"] == int(mixing_f16)
    back = fb.load_record_cache(path, host_records=host)
    ws = fb.Workspace(dh, di, K)
    for t in range(3):
        h = torch.from_numpy(O.token_input(1, t, dh)).cuda()
        for a, b in zip(layers, back):
            ta = fb.layer_forward(a, h, ws, traced=True)
            tb = fb.layer_forward(b, h, ws, traced=True)
            # u (one CTA per row), routing and masks are deterministic: identical;
            # y sums the CTAs' partials with float atomics in arrival order
            for k in ("block_input", "experts", "weights", "masks"):
                assert torch.equal(ta[k], tb[k]), k
            assert O.rel_l2(tb["out"].cpu().numpy(), ta["out"].cpu().numpy()) <= 1e-6
    for a, b in zip(layers, back):
        for ea, eb in zip(a.experts, b.experts):
            assert eb.residency()["resident"] == (not host)
            da, db = ea.download(), eb.download()
            assert all(np.array_equal(da[k], db[k]) for k in ("codes", "scales", "zeros"))
            assert da["threshold"] == db["threshold"]


def test_record_cache_errors(fb, tmp_path):
    bad = tmp_path / "bad.flor"
    bad.write_bytes(b"FLOQ" + bytes(60))
    with pytest.raises(fb.FloeError, match="record_cache: bad magic"):
        fb.record_cache_info(bad)
    bad.write_bytes(b"FLOR" + bytes(10))
    with pytest.raises(fb.FloeError, match="record_cache: truncated file"):
        fb.record_cache_info(bad)
