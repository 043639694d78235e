"""The compact record wire format (pack_compact, core/src/offload.cpp:27-53;
SURVEY §8 a12): the device packer is byte-identical to the reference's
pack_compact(element_bytes = 2) for the kept channels of a real token, and an
expert uploaded from the all-channel wire format (records_f16) computes the
same as one uploaded from f32 gate/down (test_offload.cpp:79-131: 16,384-B
records, f16 rounding once)."""
import ctypes as ct

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


@pytest.mark.parametrize("dh,di", [(4096, 2048), (2048, 512), (64, 256)])
def test_device_pack_compact_matches_reference(fb, torch, ref, dh, di):
    gate, up, down = O.seeded_expert(dh, di, 21)
    x = O.seeded_input(dh, 22)
    q = O.quantize(up, 2, 64)
    v = O.qgemv_channels(q, dh, x)
    t = O.calibrate_threshold(np.abs(v), 0.8)
    ex = O.Expert(dh, di, q, gate, down, t)
    mask = (np.abs(v) >= t).astype(np.uint8)
    want_ch, want_payload = O.pack_compact(ex, mask, 2)
    # the reference core itself (oracle/_ref) agrees with the oracle restatement
    eh = ref.ref_expert_create(dh, di, 2, 64, q.codes, q.scales, q.zeros, gate, down, t)
    assert eh
    n = int(mask.sum())
    ch_ref = np.empty(max(n, 1), np.uint32)
    pay_ref = np.empty(max(n, 1) * 4 * dh, np.uint8)
    nref = ct.c_uint64()
    assert ref.ref_pack_compact(eh, mask, 2, ch_ref, pay_ref, ct.byref(nref)) == 0
    assert nref.value == n
    ref.ref_expert_destroy(eh)
    assert np.array_equal(ch_ref[:n], want_ch) and np.array_equal(pay_ref[:n * 4 * dh], want_payload)
    assert want_payload.size == n * 4 * dh  # 16,384 B per record at d_hidden 4096
    ge = fb.GpuExpert(dh, di, 2, 64, q.codes, q.scales, q.zeros, gate=gate, down=down, threshold=t)
    ch, payload = fb.pack_compact(ge, torch.from_numpy(mask).cuda(), 2)
    assert np.array_equal(ch.cpu().numpy().astype(np.uint32), want_ch)
    assert np.array_equal(payload.cpu().numpy(), want_payload)
    with pytest.raises(fb.FloeError, match="element_bytes"):
        fb.pack_compact(ge, torch.from_numpy(mask).cuda(), 3)


def test_records_f16_wire_upload_equals_f32_upload(fb, torch):
    dh, di = 4096, 1024
    gate, up, down = O.seeded_expert(dh, di, 31)
    x = O.seeded_input(dh, 32)
    q = O.quantize(up, 2, 64)
    t = O.calibrate_threshold(np.abs(O.qgemv_channels(q, dh, x)), 0.8)
    ex = O.Expert(dh, di, q, gate, down, t)
    _, wire = O.pack_compact(ex, np.ones(di, np.uint8), 2)  # every channel, f16 wire format
    a = fb.GpuExpert(dh, di, 2, 64, q.codes, q.scales, q.zeros, gate=gate, down=down, threshold=t)
    b = fb.GpuExpert(dh, di, 2, 64, q.codes, q.scales, q.zeros, records=wire.view(np.uint16),
                     threshold=t)
    ws = fb.Workspace(dh, di)
    xd = torch.from_numpy(x).cuda()
    ya = fb.expert_forward_sparse(a, xd, ws).cpu().numpy()
    yb = fb.expert_forward_sparse(b, xd, ws).cpu().numpy()
    assert O.rel_l2(yb, ya) <= 1e-6
    assert O.rel_l2(ya, O.expert_forward_sparse(ex, x)) <= 1e-2
