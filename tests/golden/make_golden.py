"""Generate tests/golden/*.npz from the REFERENCE core (oracle/_ref/libfloe_ref.so).

Run in the dev container (where /root/reference exists and `make -C oracle`
compiled the reference sources).  The fixtures pin the C restatement
(oracle/floe_oracle.c) and the GPU path to the reference's own outputs on the
GPU box, where /root/reference is absent.  Shapes follow the reference tests:
acceptance_test.cpp:38-60 (seeded_expert / seeded_input, stream 4),
test_model.cpp:16-25 (toy_config L=2, E=4, top-2, dh=32, di=64, seed 7).

    python tests/golden/make_golden.py
"""
import ctypes as ct
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import oracle as O  # noqa: E402

R = O.REF
assert R is not None, "oracle/_ref/libfloe_ref.so missing: run `make -C oracle` here first"
OUT = Path(__file__).resolve().parent


def ref_expert(dh, di, seed):
    g, u, d = (np.empty(dh * di, np.float32) for _ in range(3))
    R.ref_seeded_expert(dh, di, seed, g, u, d)
    return g, u, d


def ref_input(dh, seed, stream=4):
    x = np.empty(dh, np.float32)
    R.ref_normals(seed, stream, dh, x)
    return x


def ref_quant(x, bits, g):
    n = x.size
    codes = np.zeros(R.ref_packed_code_bytes(n, bits), np.uint8)
    sc = np.zeros(n // g, np.uint16)
    ze = np.zeros(n // g, np.uint16)
    assert R.ref_quantize(x, n, bits, g, codes, sc, ze) == 0
    return codes, sc, ze


def expert_case(name, dh, di, seed, xseed, bits, g, k):
    gate, up, down = ref_expert(dh, di, seed)
    x = ref_input(dh, xseed)
    codes, sc, ze = ref_quant(up, bits, g)
    v = np.empty(di, np.float32)
    assert R.ref_qgemv_channels(codes, sc, ze, up.size, bits, g, dh, x, v) == 0
    t = np.float32(R.ref_calibrate_threshold(np.abs(v).astype(np.float32), di, k))
    h = R.ref_expert_create(dh, di, bits, g, codes, sc, ze, gate, down, t)
    y = np.empty(dh, np.float32)
    assert R.ref_expert_forward(h, x, y) == 0
    # the same expert with f16-rounded gate/down: what the device records hold
    gh = np.empty(gate.size, np.uint16)
    dhh = np.empty(down.size, np.uint16)
    R.ref_f32_to_f16(gate, gate.size, gh)
    R.ref_f32_to_f16(down, down.size, dhh)
    g16 = np.empty(gate.size, np.float32)
    d16 = np.empty(down.size, np.float32)
    R.ref_f16_to_f32(gh, gh.size, g16)
    R.ref_f16_to_f32(dhh, dhh.size, d16)
    h16 = R.ref_expert_create(dh, di, bits, g, codes, sc, ze, g16, d16, t)
    y16 = np.empty(dh, np.float32)
    assert R.ref_expert_forward(h16, x, y16) == 0
    deq = np.empty(up.size, np.float32)
    assert R.ref_dequantize(codes, sc, ze, up.size, bits, g, deq) == 0
    mask = (np.abs(v) >= t).astype(np.uint8)
    nch = ct.c_uint64()
    chans = np.empty(di, np.uint32)
    payload = np.empty(di * 4 * dh, np.uint8)
    assert R.ref_pack_compact(h, mask, 2, chans, payload, ct.byref(nch)) == 0
    R.ref_expert_destroy(h)
    R.ref_expert_destroy(h16)
    np.savez_compressed(
        OUT / f"{name}.npz", dh=dh, di=di, seed=seed, xseed=xseed, bits=bits, group_size=g, k=k,
        gate=gate, up=up, down=down, x=x, codes=codes, scales=sc, zeros=ze, v=v, threshold=t,
        y=y, y_f16=y16, deq=deq, mask=mask, pack_channels=chans[: nch.value],
        pack_payload=payload[: nch.value * 4 * dh])


def toy_layer_case():
    # test_model.cpp:16-25 toy_config; calibrate_model(seed 3, 64 tokens, k 0.5)
    L, E, K, dh, di = 2, 4, 2, 32, 64
    cm = R.ref_cmodel_build(L, E, K, dh, di, 7, 3, 64, 0.5, 2, 16, 1)
    assert cm, O.ref_error()
    arrays = {}
    for l in range(L):
        rp, mp = ct.POINTER(ct.c_float)(), ct.POINTER(ct.c_float)()
        R.ref_cmodel_layer_view(cm, l, ct.byref(rp), ct.byref(mp))
        arrays[f"router{l}"] = np.ctypeslib.as_array(rp, (E * dh,)).copy()
        arrays[f"mixing{l}"] = np.ctypeslib.as_array(mp, (dh * dh,)).copy()
        for e in range(E):
            h = R.ref_cmodel_expert(cm, l, e)
            c, s, z = (ct.POINTER(ct.c_uint8)(), ct.POINTER(ct.c_uint16)(),
                       ct.POINTER(ct.c_uint16)())
            gp, dp, th = ct.POINTER(ct.c_float)(), ct.POINTER(ct.c_float)(), ct.c_float()
            R.ref_expert_view(h, ct.byref(c), ct.byref(s), ct.byref(z), ct.byref(gp),
                              ct.byref(dp), ct.byref(th))
            n = dh * di
            arrays[f"codes{l}_{e}"] = np.ctypeslib.as_array(c, (n * 2 // 8,)).copy()
            arrays[f"scales{l}_{e}"] = np.ctypeslib.as_array(s, (n // 16,)).copy()
            arrays[f"zeros{l}_{e}"] = np.ctypeslib.as_array(z, (n // 16,)).copy()
            arrays[f"gate{l}_{e}"] = np.ctypeslib.as_array(gp, (n,)).copy()
            arrays[f"down{l}_{e}"] = np.ctypeslib.as_array(dp, (n,)).copy()
            arrays[f"threshold{l}_{e}"] = np.float32(th.value)
    toks = []
    for t in range(4):
        hvec = np.empty(dh, np.float32)
        R.ref_token_input(1, t, dh, hvec)
        for l in range(L):
            u = np.empty(dh, np.float32)
            sel = np.empty(K, np.uint32)
            w = np.empty(K, np.float32)
            masks = np.empty((K, di), np.uint8)
            y = np.empty(dh, np.float32)
            assert R.ref_layer_forward_traced(cm, l, hvec, u, sel, w, masks, y) == 0
            toks.append(dict(h=hvec.copy(), u=u, sel=sel, w=w, masks=masks, y=y))
            hvec = y
    for i, tk in enumerate(toks):
        for k, v in tk.items():
            arrays[f"tok{i}_{k}"] = v
    R.ref_cmodel_destroy(cm)
    np.savez_compressed(OUT / "toy_layer.npz", L=L, E=E, K=K, dh=dh, di=di, bits=2, group_size=16,
                        n_steps=len(toks), **arrays)


def scalar_cases():
    rng = np.random.default_rng(1234)
    xs = np.concatenate([rng.standard_normal(4096).astype(np.float32),
                         np.array([0.0, -0.0, 65504.0, 65520.0, 1e-8, 5.96e-8, 2.98e-8, -1e-5,
                                   np.inf, -np.inf], np.float32)])
    h = np.empty(xs.size, np.uint16)
    R.ref_f32_to_f16(xs, xs.size, h)
    allh = np.arange(65536, dtype=np.uint16)
    f = np.empty(65536, np.float32)
    R.ref_f16_to_f32(allh, 65536, f)
    n1 = np.empty(1001, np.float32)
    R.ref_normals(99, 1, 1001, n1)
    tok = np.empty(64, np.float32)
    R.ref_token_input(1, 5, 64, tok)
    logits = np.array([0.5, 2.0, 2.0, -1.0, 2.0, 0.1], np.float32)
    tk = np.empty(3, np.uint32)
    R.ref_top_k(logits, logits.size, 3, tk)
    sm = np.array([1.0, 2.0, 3.0], np.float32)
    R.ref_softmax(sm, 3)
    ratios = np.array([R.ref_compression_ratio(4096, 14336, 2, 64, 0.10, 0),
                       R.ref_compression_ratio(4096, 14336, 2, 64, 0.10, 1)])
    np.savez_compressed(OUT / "scalars.npz", f32_in=xs, f16_out=h, f16_all=f, normals_99_1=n1,
                        token_1_5=tok, topk_in=logits, topk_out=tk, softmax_out=sm,
                        ratios=ratios)


if __name__ == "__main__":
    scalar_cases()
    # acceptance check 1 shape (bits 8, g 64) and the INT2 path at small dh
    expert_case("expert_acc1_b8", 64, 256, 1000, 2000, 8, 64, 0.5)
    expert_case("expert_b2_g64", 256, 96, 11, 12, 2, 64, 0.8)
    expert_case("expert_b4_g32", 128, 64, 21, 22, 4, 32, 0.8)
    expert_case("expert_b3_g8", 32, 48, 31, 32, 3, 8, 0.8)
    expert_case("expert_b2_dh2048", 2048, 64, 41, 42, 2, 64, 0.8)
    toy_layer_case()
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size)
