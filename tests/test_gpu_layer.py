"""GPU parity of the MoE layer path (config 2) and of the device-side model
preparation (reference random streams + quantize) against the CPU oracle."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

DH, DI, E, K = 4096, 14336, 8, 2
TIE = 1e-3


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available(), "the -m gpu suite needs a CUDA device"
    return torch


@pytest.fixture(scope="module")
def fb(torch):
    import paper_2505_05950_b200 as fb
    return fb


def weight_stream(layer, kind, expert):  # core/src/model.cpp:25-28
    return ((layer * 5 + kind) * 65536 + expert) * 64


# ------------------------------------------------------- device model preparation
def test_device_normals_match_reference_streams(fb, torch):
    """floe_gpu_gen_normals == the reference Rng streams (device libm: allow a
    handful of last-ulp differences out of 58.7M values; count them)."""
    n = DH * DI
    sd = float(np.float32(1.0) / np.sqrt(np.float32(DH)))
    host = O.normals(99, 2, n, sd)                   # seeded_expert up (stream 2)
    dev = fb.gen_normals(99, 2, n, sd).cpu().numpy()
    bad = np.nonzero(host.view(np.uint32) != dev.view(np.uint32))[0]
    assert len(bad) <= 4, len(bad)
    if len(bad):
        assert np.all(np.abs(host[bad].view(np.int32) - dev[bad].view(np.int32)) <= 1)
    # gen_model's 64-shard layout
    shard = np.empty(1 << 20, np.float32)
    O.C.fo_fill_gaussian(shard, shard.size, 7, weight_stream(0, 3, 5), np.float32(sd), O.THREADS)
    devs = fb.gen_normals(7, weight_stream(0, 3, 5), 1 << 20, sd, sharded=True).cpu().numpy()
    assert np.sum(shard.view(np.uint32) != devs.view(np.uint32)) <= 1
    # token_input(1, t): Rng(1, 2^40 + t)
    assert np.array_equal(fb.gen_normals(1, (1 << 40) + 3, DH).cpu().numpy().view(np.uint32),
                          O.token_input(1, 3, DH).view(np.uint32))


@pytest.mark.parametrize("bits,g,n", [(2, 64, DH * DI), (1, 32, 4096), (3, 8, 4096),
                                      (4, 16, 4096), (8, 64, 8192), (2, 4, 4096)])
def test_device_quantize_bit_exact(fb, torch, bits, g, n):
    x = O.normals(11, 3, n, 0.02)
    q = O.quantize(x, bits, g)
    codes, scales, zeros = fb.quantize(torch.from_numpy(x).cuda(), bits, g)
    assert np.array_equal(codes.cpu().numpy(), q.codes)
    assert np.array_equal(scales.cpu().numpy().view(np.uint16), q.scales)
    assert np.array_equal(zeros.cpu().numpy().view(np.uint16), q.zeros)


# ------------------------------------------------------------------ toy layer
def test_toy_layer_matches_golden(fb, torch, golden):
    """test_model.cpp toy_config (L=2, E=4, top-2, dh=32, di=64): the generic
    kernels against the reference's layer_forward_traced outputs."""
    g = golden("toy_layer")
    L, En, Kk, dh, di = (int(g[k]) for k in ("L", "E", "K", "dh", "di"))
    layers = []
    keep = []
    for l in range(L):
        ex = [fb.GpuExpert(dh, di, 2, 16, g[f"codes{l}_{e}"], g[f"scales{l}_{e}"],
                           g[f"zeros{l}_{e}"], gate=g[f"gate{l}_{e}"], down=g[f"down{l}_{e}"],
                           threshold=float(g[f"threshold{l}_{e}"])) for e in range(En)]
        keep.append(ex)
        layers.append(fb.GpuLayer(g[f"router{l}"].reshape(En, dh), g[f"mixing{l}"].reshape(dh, dh),
                                  ex, Kk, mixing_f16=False))
    ws = fb.Workspace(dh, di, Kk)
    for i in range(int(g["n_steps"])):
        tr = fb.layer_forward(layers[i % L], torch.from_numpy(g[f"tok{i}_h"]).cuda(), ws,
                              traced=True)
        torch.cuda.synchronize()
        u = tr["block_input"].cpu().numpy()
        assert O.rel_l2(u, g[f"tok{i}_u"]) <= 1e-6
        assert np.array_equal(tr["experts"].cpu().numpy(), g[f"tok{i}_sel"].astype(np.int32))
        assert np.allclose(tr["weights"].cpu().numpy(), g[f"tok{i}_w"], rtol=1e-5, atol=1e-6)
        masks = tr["masks"].cpu().numpy()
        assert np.array_equal(masks, g[f"tok{i}_masks"])
        assert O.rel_l2(tr["out"].cpu().numpy(), g[f"tok{i}_y"]) <= 1e-3


# ------------------------------------------------------------- Mixtral layer
@pytest.fixture(scope="module")
def mixtral_layer():
    """One gen_model layer (seed 7) at Mixtral shape, built by the oracle on the
    host; thresholds = calibrate_threshold(|qgemv(up_e, u_cal)|, 0.8) on the
    block input of token_input(3, 0)."""
    sd = np.float32(1.0) / np.sqrt(np.float32(DH))

    def fill(kind, e, n):
        out = np.empty(n, np.float32)
        O.C.fo_fill_gaussian(out, n, 7, weight_stream(0, kind, e), sd, O.THREADS)
        return out

    router = fill(0, 0, E * DH).reshape(E, DH)
    mixing = fill(1, 0, DH * DH).reshape(DH, DH)
    h_cal = O.token_input(3, 0, DH)
    mixed = np.empty(DH, np.float32)
    O.C.fo_gemv(DH, DH, mixing, h_cal, mixed)
    u_cal = h_cal + mixed
    experts = []
    for e in range(E):
        gate, up, down = fill(2, e, DH * DI), fill(3, e, DH * DI), fill(4, e, DH * DI)
        q = O.quantize(up, 2, 64)
        t = O.calibrate_threshold(np.abs(O.qgemv_channels(q, DH, u_cal)), 0.8)
        experts.append(O.Expert(DH, DI, q, gate, down, t))
    return O.Layer(router, mixing, experts, K)


def upload_layer(fb, L, mixing_f16):
    ex = [fb.GpuExpert(DH, DI, 2, 64, e.up_q.codes, e.up_q.scales, e.up_q.zeros, gate=e.gate,
                       down=e.down_t, threshold=e.threshold) for e in L.experts]
    return fb.GpuLayer(L.router, L.mixing, ex, K, mixing_f16=mixing_f16)


def test_mixtral_layer_parity(fb, torch, mixtral_layer):
    L = mixtral_layer
    gl = upload_layer(fb, L, mixing_f16=False)
    ws = fb.Workspace(DH, DI, K)
    for t in range(3):
        h = O.token_input(1, t, DH)
        ref = O.layer_forward(L, h, traced=True)
        tr = fb.layer_forward(gl, torch.from_numpy(h).cuda(), ws, traced=True)
        torch.cuda.synchronize()
        u = tr["block_input"].cpu().numpy()
        assert O.rel_l2(u, ref["block_input"]) <= 1e-6
        assert np.array_equal(tr["experts"].cpu().numpy(), ref["experts"].astype(np.int32))
        assert np.allclose(tr["weights"].cpu().numpy(), ref["weights"], rtol=1e-5)
        masks = tr["masks"].cpu().numpy()
        for j, e in enumerate(ref["experts"]):
            v = O.qgemv_channels(L.experts[e].up_q, DH, ref["block_input"])
            diff = np.nonzero(masks[j] != ref["masks"][j])[0]
            assert np.all(np.abs(np.abs(v[diff]) - L.experts[e].threshold) <= TIE)
        assert O.rel_l2(tr["out"].cpu().numpy(), ref["out"]) <= 1e-2


def test_mixtral_layer_f16_mixing_and_host_call(fb, torch, mixtral_layer):
    L = mixtral_layer
    gl = upload_layer(fb, L, mixing_f16=True)
    ws = fb.Workspace(DH, DI, K)
    for t in range(3, 6):
        h = O.token_input(1, t, DH)
        ref = O.layer_forward(L, h)
        y = fb.layer_forward(gl, torch.from_numpy(h).cuda(), ws).cpu().numpy()
        assert O.rel_l2(y, ref) <= 1e-2
        yh = fb.layer_forward_host(gl, h, ws)
        assert O.rel_l2(yh, y) <= 1e-6
    c0 = ws.read_counters()
    ws.reset_counters()
    for t in range(4):
        fb.layer_forward(gl, torch.from_numpy(O.token_input(1, t, DH)).cuda(), ws)
    c = ws.read_counters()
    assert c["calls"] == 4 and 0.15 * 4 * K * DI < c["kept"] < 0.25 * 4 * K * DI
    assert c0["calls"] >= 6
