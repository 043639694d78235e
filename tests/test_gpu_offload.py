"""Host-resident gate|down records (SURVEY config 3, ExpertCache residency of
core/src/offload.cpp:89-159 at expert granularity): the kernels read the kept
channels' records in place from pinned host memory over PCIe; promotion to
HBM and demotion are stream-ordered and switch every layer table holding the
expert.  Outputs must not depend on where the records live."""
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


@pytest.mark.parametrize("dh,di,bits,g", [(4096, 2048, 2, 64), (2048, 512, 2, 64), (64, 256, 8, 64)])
def test_expert_forward_independent_of_residency(fb, torch, dh, di, bits, g):
    gate, up, down = O.seeded_expert(dh, di, 5)
    x = O.seeded_input(dh, 6)
    q = O.quantize(up, bits, g)
    t = O.calibrate_threshold(np.abs(O.qgemv_channels(q, dh, x)), 0.8)
    dev = fb.GpuExpert(dh, di, bits, g, q.codes, q.scales, q.zeros, gate=gate, down=down,
                       threshold=t)
    host = fb.GpuExpert(dh, di, bits, g, q.codes, q.scales, q.zeros, gate=gate, down=down,
                        threshold=t, host_records=True)
    assert host.residency() == dict(resident=False, device_bytes=0)
    ws = fb.Workspace(dh, di)
    xd = torch.from_numpy(x).cuda()
    y_dev = fb.expert_forward_sparse(dev, xd, ws).cpu().numpy()
    y_host = fb.expert_forward_sparse(host, xd, ws).cpu().numpy()
    assert O.rel_l2(y_host, y_dev) <= 1e-6
    # promote, demote, promote: same result each time
    for r in (True, False, True):
        host.set_resident(r)
        assert host.residency()["resident"] == r
        y = fb.expert_forward_sparse(host, xd, ws).cpu().numpy()
        assert O.rel_l2(y, y_dev) <= 1e-6


def test_layer_tables_follow_residency(fb, torch):
    dh, di, E, K = 2048, 512, 4, 2
    rng = np.random.default_rng(3)
    experts, hosted = [], []
    for e in range(E):
        gate, up, down = O.seeded_expert(dh, di, 40 + e)
        q = O.quantize(up, 2, 64)
        experts.append(fb.GpuExpert(dh, di, 2, 64, q.codes, q.scales, q.zeros, gate=gate,
                                    down=down, threshold=1.0))
        hosted.append(fb.GpuExpert(dh, di, 2, 64, q.codes, q.scales, q.zeros, gate=gate,
                                   down=down, threshold=1.0, host_records=True))
    router = (rng.standard_normal((E, dh)) / 45).astype(np.float32)
    mixing = (rng.standard_normal((dh, dh)) / 45).astype(np.float32)
    la = fb.GpuLayer(router, mixing, experts, K)
    lb = fb.GpuLayer(router, mixing, hosted, K)
    ws = fb.Workspace(dh, di, K)
    for t in range(3):
        h = torch.from_numpy(O.token_input(1, t, dh)).cuda()
        ya = fb.layer_forward(la, h, ws).cpu().numpy()
        yb = fb.layer_forward(lb, h, ws).cpu().numpy()
        assert O.rel_l2(yb, ya) <= 1e-6
        hosted[t % E].set_resident(True)  # the layer table switches with the expert
        yc = fb.layer_forward(lb, h, ws).cpu().numpy()
        assert O.rel_l2(yc, ya) <= 1e-6


def _stack(fb, L, E, K, dh, di, host):
    rng = np.random.default_rng(11)
    layers = []
    for l in range(L):
        ex = []
        for e in range(E):
            gate, up, down = O.seeded_expert(dh, di, 100 * l + e)
            q = O.quantize(up, 2, 64)
            ex.append(fb.GpuExpert(dh, di, 2, 64, q.codes, q.scales, q.zeros, gate=gate,
                                   down=down, threshold=1.0, host_records=host))
        router = (rng.standard_normal((E, dh)) / 45).astype(np.float32)
        mixing = (rng.standard_normal((dh, dh)) / 45).astype(np.float32)
        layers.append(fb.GpuLayer(router, mixing, ex, K))
    return layers


@pytest.mark.parametrize("budget_experts", [0, 3, 100])
def test_offload_decode_matches_resident_chain(fb, torch, budget_experts):
    """decode through host-resident layers == the chain of layer_forward calls
    on HBM-resident copies, for any VRAM budget; the record accounting covers
    every kept channel exactly once."""
    L, E, K, dh, di = 3, 4, 2, 2048, 512
    ref_layers = _stack(fb, L, E, K, dh, di, host=False)
    host_layers = _stack(fb, L, E, K, dh, di, host=True)
    off = fb.Offload(host_layers, budget_experts * 4 * dh * di)
    ws = fb.Workspace(dh, di, K)
    ws_ref = fb.Workspace(dh, di, K)
    ws_ref.reset_counters()
    for t in range(6):
        h = torch.from_numpy(O.token_input(2, t, dh)).cuda()
        y = off.decode(h, ws)
        r = h
        for L_ in ref_layers:
            r = fb.layer_forward(L_, r, ws_ref)
        torch.cuda.synchronize()
        assert O.rel_l2(y.cpu().numpy(), r.cpu().numpy()) <= 1e-5
    st = off.stats()
    kept = ws_ref.read_counters()["kept"]
    assert st["tokens"] == 6
    assert st["records_from_hbm"] + st["records_over_pcie"] == kept
    if budget_experts == 0:
        assert st["records_from_hbm"] == 0 and st["promotions"] == 0
    if budget_experts == 100:
        assert st["promotions"] > 0 and st["evictions"] == 0
        assert st["records_from_hbm"] > 0
    assert st["device_record_bytes"] <= budget_experts * 4 * dh * di
    off.close()


def test_offload_decode_replay_matches_layer_forward(fb, torch):
    """decode_replay: layer l on its own recorded block input == layer_forward."""
    L, E, K, dh, di = 3, 4, 2, 2048, 512
    ref_layers = _stack(fb, L, E, K, dh, di, host=False)
    off = fb.Offload(_stack(fb, L, E, K, dh, di, host=True), 2 * 4 * dh * di)
    ws, ws_ref = fb.Workspace(dh, di, K), fb.Workspace(dh, di, K)
    for t in range(4):
        h = torch.stack([torch.from_numpy(O.token_input(7 + l, t, dh)) for l in range(L)]).cuda()
        y = off.decode_replay(h, ws)
        for l in range(L):
            r = fb.layer_forward(ref_layers[l], h[l], ws_ref)
            assert O.rel_l2(y[l].cpu().numpy(), r.cpu().numpy()) <= 1e-5
    with pytest.raises(fb.FloeError):
        off.decode_replay(h[0], ws)
    off.close()


@pytest.mark.parametrize("dh,di", [(4096, 2048), (2048, 512), (256, 256)])
@pytest.mark.parametrize("bad", ["inf", "nan"])
def test_layer_forward_nonfinite_input_terminates(fb, torch, dh, di, bad):
    """A non-finite block input (a random-weight stack chained far enough
    overflows) must give an in-range routing and a non-finite output, never a
    hang or a fault.  The reference's top_k comparator (la.cpp:52-55) is not a
    strict weak order with NaNs; here NaN ranks below every number."""
    E, K = 4, 2
    ex = []
    for e in range(E):
        gate, up, down = O.seeded_expert(dh, di, 300 + e)
        q = O.quantize(up, 2, 64)
        ex.append(fb.GpuExpert(dh, di, 2, 64, q.codes, q.scales, q.zeros, gate=gate, down=down,
                               threshold=1.0))
    rng = np.random.default_rng(5)
    router = (rng.standard_normal((E, dh)) / np.sqrt(dh)).astype(np.float32)
    mixing = (rng.standard_normal((dh, dh)) / np.sqrt(dh)).astype(np.float32)
    layer = fb.GpuLayer(router, mixing, ex, K)
    ws = fb.Workspace(dh, di, K)
    h = torch.from_numpy(O.token_input(1, 0, dh)).cuda()
    h[dh // 3] = float(bad)
    r = fb.layer_forward(layer, h, ws, traced=True)
    torch.cuda.synchronize()
    sel = r["experts"].cpu().numpy()
    assert ((sel >= 0) & (sel < E)).all() and len(set(sel.tolist())) == K
    assert list(sel) == sorted(sel)
    assert not torch.isfinite(r["out"]).all()
    # the device is still healthy: a finite input afterwards gives the normal result
    h2 = torch.from_numpy(O.token_input(1, 1, dh)).cuda()
    y2 = fb.layer_forward(layer, h2, ws).cpu().numpy()
    assert np.isfinite(y2).all()
