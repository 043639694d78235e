"""Offload engine accounting and predictor scoring.

* DecodeTimeline identities (core/include/floe/offload.hpp:128-157):
  demanded == from_cache + prefetch_used + sync, and every byte moved is
  prefetch_used + prefetch_wasted + sync (+ promotions not yet resolved),
  cross-checked against the kernel's own HBM / PCIe record counters.
* eval_masks / eval_sets (core/src/predictor.cpp:206-254) on the decode path:
  the engine's scores equal the same metrics recomputed here from traced
  layer_forward calls, predict_mask and predict_experts."""
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


def _stack(fb, L, E, K, dh, di, host, seed=11):
    rng = np.random.default_rng(seed)
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
def test_timeline_identities(fb, torch, budget_experts):
    L, E, K, dh, di = 4, 4, 2, 2048, 512
    off = fb.Offload(_stack(fb, L, E, K, dh, di, host=True), budget_experts * 4 * dh * di)
    ws = fb.Workspace(dh, di, K)
    T = 10
    for t in range(T):
        h = torch.stack([torch.from_numpy(O.token_input(3 + l, t % 5, dh)) for l in range(L)]).cuda()
        off.decode_replay(h, ws)
    st = off.stats()
    rb = st["record_bytes"]
    ups = T * L * K * st["up_bytes_per_expert"]
    assert st["tokens"] == T
    # every demanded byte lands in exactly one bucket
    assert st["bytes_demanded"] == st["bytes_from_cache"] + st["bytes_prefetch_used"] + st["bytes_sync"]
    # every moved byte is used, wasted, sync, or a promotion still unresolved
    moved = st["bytes_promoted"] + st["bytes_sync"]
    assert moved == (st["bytes_prefetch_used"] + st["bytes_prefetch_wasted"] + st["bytes_sync"]
                     + st["bytes_prefetch_pending"])
    # the classification agrees with the kernel's per-record placement counters
    assert st["bytes_sync"] == st["records_over_pcie"] * rb
    assert st["bytes_demanded"] - ups == (st["records_from_hbm"] + st["records_over_pcie"]) * rb
    assert st["bytes_from_cache"] + st["bytes_prefetch_used"] - ups == st["records_from_hbm"] * rb
    assert st["requests_channel"] == st["records_over_pcie"] + st["promotions"]
    if budget_experts == 0:
        assert st["bytes_prefetch_used"] == 0 and st["bytes_promoted"] == 0
        assert st["bytes_sync"] == st["bytes_demanded"] - ups
    if budget_experts == 100:
        assert st["promotions"] > 0 and st["bytes_prefetch_used"] > 0
        assert st["bytes_prefetch_wasted"] > 0  # a promotion moves the whole record block
    off.close()


def _pr(pred, truth):
    inter = len(set(pred) & set(truth))
    p = (1.0 if not truth else 0.0) if not pred else inter / len(pred)
    r = 1.0 if not truth else inter / len(truth)
    return p, r


@pytest.mark.parametrize("replay", [True, False])
def test_eval_scores_match_recomputed(fb, torch, replay):
    """The engine's mask / set precision and recall == eval_masks / eval_sets
    of predict_mask(layer l expert, u_{l-1}) and predict_experts(u_{l-1})
    against the routed experts and their true masks, recomputed from traced
    layer_forward calls on HBM-resident copies of the same stack."""
    L, E, K, dh, di = 4, 4, 2, 2048, 512
    ref = _stack(fb, L, E, K, dh, di, host=False)
    off = fb.Offload(_stack(fb, L, E, K, dh, di, host=True), 2 * 4 * dh * di)
    rng = np.random.default_rng(5)
    w = (rng.standard_normal((L - 1, E, dh)) / 45).astype(np.float32)
    b = (rng.standard_normal((L - 1, E)) * 0.1).astype(np.float32)
    pred = fb.GpuPredictor(w, b)
    off.set_eval(True, pred, 2)
    ws, ws_r = fb.Workspace(dh, di, K), fb.Workspace(dh, di, K)
    mp, mr, sp, sr, ns, nm = 0.0, 0.0, 0.0, 0.0, 0, 0
    for t in range(3):
        hs = torch.stack([torch.from_numpy(O.token_input(9 + l, t, dh)) for l in range(L)]).cuda()
        if replay:
            off.decode_replay(hs, ws)
        else:
            off.decode(hs[0], ws)
        h = hs[0]
        prev_u = None
        for l in range(L):
            tr = fb.layer_forward(ref[l], hs[l] if replay else h, ws_r, traced=True)
            sel = tr["experts"].cpu().numpy().tolist()
            masks = tr["masks"].cpu().numpy()
            if l > 0:
                for k, e in enumerate(sel):
                    pm = fb.predict_mask(ref[l].experts[e], prev_u, ref[l].experts[e].threshold,
                                         ws_r).cpu().numpy()
                    p, r = _pr(np.nonzero(pm)[0].tolist(), np.nonzero(masks[k])[0].tolist())
                    mp, mr, nm = mp + p, mr + r, nm + 1
                ps = fb.predict_experts(pred, prev_u, l, 2).cpu().numpy().tolist()
                p, r = _pr(ps, sel)
                sp, sr, ns = sp + p, sr + r, ns + 1
            prev_u = tr["block_input"].clone()
            h = tr["out"]
    st = off.stats()
    assert st["mask_samples"] == nm and st["set_samples"] == ns
    assert abs(st["mask_precision"] - mp / nm) <= 1e-9
    assert abs(st["mask_recall"] - mr / nm) <= 1e-9
    assert abs(st["set_precision"] - sp / ns) <= 1e-9
    assert abs(st["set_recall"] - sr / ns) <= 1e-9
    off.close()
