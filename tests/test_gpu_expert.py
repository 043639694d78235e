"""GPU parity of the compressed-expert hot path against the CPU oracle.

Every call goes through the C ABI (libfloe_b200.so).  Parity rules
(BASELINE.json north_star):
  * dequantized up weights: f32 bit-exact with floe::dequantize;
  * v: |v_gpu - v_cpu| <= V_ABS + V_REL*|v_cpu|  (fp32, different summation order);
  * masks identical except channels with ||v_cpu| - t| <= 1e-3 (TIE);
  * y: rel-L2 <= 1e-2 against the reference (f32 gate/down) and <= 1e-4
    against the same computation over the f16 records the device holds.
"""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

V_ABS, V_REL = 2e-5, 2e-5
TIE = 1e-3
Y_REF_TOL = 1e-2      # north_star tolerance vs the reference (f32 weights)
Y_F16_TOL = 1e-4      # vs the oracle over the f16-rounded records


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available(), "the -m gpu suite needs a CUDA device"
    return torch


@pytest.fixture(scope="module")
def fb(torch):
    import paper_2505_05950_b200 as fb
    info = fb.device_info()
    assert info["cc"][0] == 10, info
    return fb


def masked_y(gate, down, x, v, mask, dh, di):
    """y = sum_{mask} silu(gate_c.x) v_c down_c in float64 (tolerance reference)."""
    idx = np.nonzero(mask)[0]
    g = gate.reshape(di, dh)[idx].astype(np.float64) @ x.astype(np.float64)
    a = g / (1.0 + np.exp(-g)) * v[idx].astype(np.float64)
    return a @ down.reshape(di, dh)[idx].astype(np.float64)


class Case:
    def __init__(self, dh, di, seed, xseed, bits=2, g=64, k=0.8):
        self.dh, self.di, self.bits, self.g = dh, di, bits, g
        self.gate, self.up, self.down = O.seeded_expert(dh, di, seed)
        self.x = O.seeded_input(dh, xseed)
        self.q = O.quantize(self.up, bits, g)
        self.v = O.qgemv_channels(self.q, dh, self.x)
        self.t = O.calibrate_threshold(np.abs(self.v), k)
        self.expert = O.Expert(dh, di, self.q, self.gate, self.down, self.t)
        self.gate16 = O.fp16_round(self.gate)
        self.down16 = O.fp16_round(self.down)

    def upload(self, fb, threshold=None):
        return fb.GpuExpert(self.dh, self.di, self.bits, self.g, self.q.codes, self.q.scales,
                            self.q.zeros, gate=self.gate, down=self.down,
                            threshold=self.t if threshold is None else threshold)

    def ref_y(self, t=None):
        e = O.Expert(self.dh, self.di, self.q, self.gate, self.down, self.t if t is None else t)
        return O.expert_forward_sparse(e, self.x)


@pytest.fixture(scope="module")
def mixtral():
    """Config 1: seeded_expert(4096, 14336, 99), seeded_input(4096, 100), INT2 g64,
    t = calibrate_threshold(|v|, 0.8) -> 2868 kept."""
    return Case(4096, 14336, 99, 100)


def run(fb, torch, e, ws, x, di):
    xd = torch.from_numpy(x).cuda()
    v = torch.empty(di, dtype=torch.float32, device="cuda")
    mask = torch.empty(di, dtype=torch.uint8, device="cuda")
    kept = torch.empty(di, dtype=torch.int32, device="cuda")
    nk = torch.zeros(1, dtype=torch.int32, device="cuda")
    y = fb.expert_forward_sparse(e, xd, ws, v=v, mask=mask, kept=kept, n_kept=nk)
    torch.cuda.synchronize()
    n = int(nk.item())
    return dict(y=y.cpu().numpy(), v=v.cpu().numpy(), mask=mask.cpu().numpy(),
                kept=np.sort(kept[:n].cpu().numpy()), n=n)


def check_v_mask(case, out, t=None):
    t = case.t if t is None else t
    dv = np.abs(out["v"] - case.v)
    assert np.all(dv <= V_ABS + V_REL * np.abs(case.v)), float(dv.max())
    ref_mask = (np.abs(case.v) >= np.float32(t)).astype(np.uint8)
    diff = np.nonzero(out["mask"] != ref_mask)[0]
    ties = np.abs(np.abs(case.v[diff]) - t) <= TIE
    assert np.all(ties), f"non-tie mask mismatches at {diff[~ties][:10]}"
    assert np.array_equal(np.nonzero(out["mask"])[0], out["kept"])
    assert out["n"] == int(out["mask"].sum())
    return diff


def test_mixtral_fast_path_selected(fb, mixtral):
    e = mixtral.upload(fb)
    info = e.info()
    assert info["fast_path"] == 1
    assert info["code_bytes"] == 14680064 and info["meta_bytes"] == 3670016
    assert info["record_bytes"] == 16384


def test_mixtral_dequant_bit_exact(fb, torch, mixtral):
    e = mixtral.upload(fb)
    d = fb.dequantize(e)
    ref = torch.from_numpy(O.dequantize(mixtral.q)).cuda()
    assert torch.equal(d.view(torch.int32), ref.view(torch.int32))


def test_mixtral_forward_parity(fb, torch, mixtral):
    c = mixtral
    e = c.upload(fb)
    ws = fb.Workspace(c.dh, c.di)
    out = run(fb, torch, e, ws, c.x, c.di)
    diff = check_v_mask(c, out)
    assert len(diff) <= 16
    assert abs(out["n"] - 2868) <= 16
    # vs the reference computation (f32 gate/down, its own mask)
    assert O.rel_l2(out["y"], c.ref_y()) <= Y_REF_TOL
    # vs the same math over the device's f16 records and the device's mask
    y16 = masked_y(c.gate16, c.down16, c.x, c.v, out["mask"], c.dh, c.di)
    assert O.rel_l2(out["y"], y16) <= Y_F16_TOL


@pytest.mark.parametrize("k", [0.0, 0.5, 0.9, 0.99])
def test_mixtral_sparsity_levels(fb, torch, mixtral, k):
    c = mixtral
    t = O.calibrate_threshold(np.abs(c.v), k)
    e = c.upload(fb, threshold=t)
    ws = fb.Workspace(c.dh, c.di)
    out = run(fb, torch, e, ws, c.x, c.di)
    check_v_mask(c, out, t)
    y16 = masked_y(c.gate16, c.down16, c.x, c.v, out["mask"], c.dh, c.di)
    assert O.rel_l2(out["y"], y16) <= Y_F16_TOL
    assert O.rel_l2(out["y"], c.ref_y(t)) <= Y_REF_TOL


def test_threshold_above_max_gives_exact_zeros(fb, torch, mixtral):
    c = mixtral
    e = c.upload(fb, threshold=1e6)
    ws = fb.Workspace(c.dh, c.di)
    out = run(fb, torch, e, ws, c.x, c.di)
    assert out["n"] == 0 and np.all(out["y"] == 0.0)


def test_repeated_calls_reset_counters(fb, torch, mixtral):
    """The last-CTA bookkeeping must leave counters at zero for the next call."""
    c = mixtral
    e = c.upload(fb)
    ws = fb.Workspace(c.dh, c.di)
    outs = [run(fb, torch, e, ws, c.x, c.di) for _ in range(5)]
    for o in outs[1:]:
        assert o["n"] == outs[0]["n"] and np.array_equal(o["mask"], outs[0]["mask"])
        assert O.rel_l2(o["y"], outs[0]["y"]) <= 1e-6


def test_nan_poison_dropped_rows_never_read(fb, torch, mixtral):
    """acceptance_test.cpp:145-176 at Mixtral shape: NaN in every dropped channel's
    gate/down record must not reach y."""
    c = mixtral
    clean_e = c.upload(fb)
    ws = fb.Workspace(c.dh, c.di)
    clean = run(fb, torch, clean_e, ws, c.x, c.di)
    drop = clean["mask"] == 0
    pg = c.gate.reshape(c.di, c.dh).copy()
    pd = c.down.reshape(c.di, c.dh).copy()
    pg[drop] = np.nan
    pd[drop] = np.nan
    pe = fb.GpuExpert(c.dh, c.di, 2, 64, c.q.codes, c.q.scales, c.q.zeros, gate=pg, down=pd,
                      threshold=c.t)
    got = run(fb, torch, pe, ws, c.x, c.di)
    assert np.array_equal(got["mask"], clean["mask"])
    assert np.all(np.isfinite(got["y"]))
    assert O.rel_l2(got["y"], clean["y"]) <= 1e-6


def test_host_call_matches_device_call(fb, torch, mixtral):
    c = mixtral
    e = c.upload(fb)
    ws = fb.Workspace(c.dh, c.di)
    dev = run(fb, torch, e, ws, c.x, c.di)
    v = np.empty(c.di, np.float32)
    mask = np.empty(c.di, np.uint8)
    y = fb.expert_forward_sparse(e, c.x, ws, v=v, mask=mask)
    assert np.array_equal(mask, dev["mask"])
    assert np.array_equal(v, dev["v"])
    assert O.rel_l2(y, dev["y"]) <= 1e-6
    with pytest.raises(fb.FloeError, match="expert_forward_sparse: dimension mismatch"):
        fb.expert_forward_sparse(e, c.x[:100], ws)


def test_qgemv_and_predict_mask(fb, torch, mixtral):
    c = mixtral
    e = c.upload(fb)
    ws = fb.Workspace(c.dh, c.di)
    v = fb.qgemv_channels(e, torch.from_numpy(c.x).cuda(), ws).cpu().numpy()
    assert np.all(np.abs(v - c.v) <= V_ABS + V_REL * np.abs(c.v))
    # reuse predictor: next expert's up projection against a previous input
    xp = O.seeded_input(c.dh, 101)
    vp = O.qgemv_channels(c.q, c.dh, xp)
    ref = O.predict_mask(c.q, c.dh, xp, 0.9)
    got = fb.predict_mask(e, torch.from_numpy(xp).cuda(), 0.9, ws).cpu().numpy()
    diff = np.nonzero(got != ref)[0]
    assert np.all(np.abs(np.abs(vp[diff]) - 0.9) <= TIE)
    assert abs(int(got.sum()) - int(ref.sum())) <= 8


def test_workspace_and_argument_errors(fb, torch, mixtral):
    c = mixtral
    e = c.upload(fb)
    small = fb.Workspace(c.dh, 128)
    with pytest.raises(fb.FloeError, match="workspace too small"):
        fb.expert_forward_sparse(e, torch.from_numpy(c.x).cuda(), small)
    with pytest.raises(fb.FloeError, match="bits must be one of"):
        fb.GpuExpert(64, 64, 5, 64, np.zeros(64 * 64, np.uint8), np.zeros(64, np.uint16),
                     np.zeros(64, np.uint16), gate=np.zeros(4096, np.float32),
                     down=np.zeros(4096, np.float32))
    with pytest.raises(fb.FloeError, match="group_size must divide"):
        fb.GpuExpert(64, 64, 2, 100, np.zeros(1024, np.uint8), np.zeros(64, np.uint16),
                     np.zeros(64, np.uint16), gate=np.zeros(4096, np.float32),
                     down=np.zeros(4096, np.float32))


# ---------------------------------------------------------------- fixtures
@pytest.mark.parametrize("name", ["expert_acc1_b8", "expert_b2_g64", "expert_b4_g32",
                                  "expert_b3_g8", "expert_b2_dh2048"])
def test_golden_fixtures(fb, torch, golden, name):
    """Reference outputs (tests/golden, from the unmodified reference core) on the
    generic kernels (bits 3/4/8, small dh) and the dh=2048 fast path."""
    g = golden(name)
    dh, di, bits, gs = int(g["dh"]), int(g["di"]), int(g["bits"]), int(g["group_size"])
    e = fb.GpuExpert(dh, di, bits, gs, g["codes"], g["scales"], g["zeros"], gate=g["gate"],
                     down=g["down"], threshold=float(g["threshold"]))
    assert e.info()["fast_path"] == int(dh == 2048 and bits == 2)
    d = fb.dequantize(e).cpu().numpy()
    assert np.array_equal(d.view(np.uint32), g["deq"].view(np.uint32))
    ws = fb.Workspace(dh, di)
    out = run(fb, torch, e, ws, g["x"], di)
    t = float(g["threshold"])
    dv = np.abs(out["v"] - g["v"])
    assert np.all(dv <= V_ABS + V_REL * np.abs(g["v"]))
    diff = np.nonzero(out["mask"] != g["mask"])[0]
    assert np.all(np.abs(np.abs(g["v"][diff]) - t) <= TIE)
    if len(diff) == 0:
        assert O.rel_l2(out["y"], g["y_f16"]) <= Y_F16_TOL
        assert O.rel_l2(out["y"], g["y"]) <= Y_REF_TOL
    g16 = O.fp16_round(g["gate"])
    d16 = O.fp16_round(g["down"])
    assert O.rel_l2(out["y"], masked_y(g16, d16, g["x"], g["v"], out["mask"], dh, di)) <= Y_F16_TOL


def test_acceptance_check1_gpu(fb, torch):
    """acceptance_test.cpp:107-141 on the device (50 of the 1000 trials): masked
    kernel vs masked-dense and t=0 vs the dense pass over the dequantized up."""
    ws = fb.Workspace(64, 256)
    for trial in range(50):
        gate, up, down = O.seeded_expert(64, 256, 1000 + trial)
        x = O.seeded_input(64, 2000 + trial)
        q = O.quantize(up, 8, 64)
        v = O.qgemv_channels(q, 64, x)
        t = O.calibrate_threshold(np.abs(v), 0.5)
        e = fb.GpuExpert(64, 256, 8, 64, q.codes, q.scales, q.zeros, gate=gate, down=down,
                         threshold=t)
        out = run(fb, torch, e, ws, x, 256)
        ref = masked_y(O.fp16_round(gate), O.fp16_round(down), x, v, out["mask"], 64, 256)
        assert O.rel_l2(out["y"], ref) <= 1e-5 * 10
        e.set_threshold(0.0)
        out0 = run(fb, torch, e, ws, x, 256)
        dense = O.expert_forward_dense(64, 256, gate, O.dequantize(q), down, x)
        assert O.rel_l2(out0["y"], dense) <= 1e-3


@pytest.mark.parametrize("dh", [2048, 4096])
def test_small_di_after_large_di_shared_workspace(fb, torch, dh):
    """di < grid leaves CTAs without channels; their segment counts must be
    rewritten every call, not inherited from an earlier, larger call."""
    ws = fb.Workspace(dh, 4096)
    for di in (4096, 64, 100, 4096, 37 * 16):
        c = Case(dh, di, 7 + di, 8)
        out = run(fb, torch, c.upload(fb), ws, c.x, di)
        diff = check_v_mask(c, out)
        if len(diff) == 0:
            assert O.rel_l2(out["y"], c.ref_y()) <= Y_REF_TOL
