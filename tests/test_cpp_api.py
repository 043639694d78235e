"""The C++ value-type API (include/floe_b200.hpp) against the reference core.

CPU: the header compiles and links against libfloe_b200.so.
GPU: tests/cpp/test_api.cpp loads a FLOQ file written by the reference's own
save_compressed (model.cpp:414-432) with floe::gpu::load_compressed, runs the
decode chain and the expert/predictor calls on the device, and every output
is compared with the reference (oracle/_ref) on the same inputs.
"""
import ctypes as ct
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O

ROOT = Path(__file__).resolve().parents[1]
LIBDIR = ROOT / "paper_2505_05950_b200"


def _ref_view(ref, eh, dh, di):
    n = dh * di
    c, sc, z = ct.POINTER(ct.c_uint8)(), ct.POINTER(ct.c_uint16)(), ct.POINTER(ct.c_uint16)()
    g, d, t = ct.POINTER(ct.c_float)(), ct.POINTER(ct.c_float)(), ct.c_float()
    ref.ref_expert_view(eh, ct.byref(c), ct.byref(sc), ct.byref(z), ct.byref(g), ct.byref(d),
                        ct.byref(t))
    codes = np.ctypeslib.as_array(c, shape=(n // 4,)).copy()
    scales = np.ctypeslib.as_array(sc, shape=(n // 64,)).copy()
    zeros = np.ctypeslib.as_array(z, shape=(n // 64,)).copy()
    return codes, scales, zeros, t.value


def _ref_qgemv(ref, eh, dh, di, x):
    codes, scales, zeros, _ = _ref_view(ref, eh, dh, di)
    v = np.empty(di, np.float32)
    assert ref.ref_qgemv_channels(codes, scales, zeros, dh * di, 2, 64, dh,
                                  np.ascontiguousarray(x, np.float32), v) == 0
    return v


def _ref_threshold(ref, eh, dh, di):
    return _ref_view(ref, eh, dh, di)[3]


def build(tmp: Path) -> Path:
    exe = tmp / "test_api"
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", f"-I{ROOT / 'include'}",
                    str(ROOT / "tests" / "cpp" / "test_api.cpp"), f"-L{LIBDIR}", "-lfloe_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", str(exe)], check=True, capture_output=True)
    return exe


def test_cpp_api_compiles_and_links(tmp_path):
    exe = build(tmp_path)
    assert exe.exists()


@pytest.mark.gpu
@pytest.mark.parametrize("dh,di", [(2048, 512), (64, 256)])
def test_cpp_api_matches_reference(tmp_path, ref, dh, di):
    L, E, K = 2, 4, 2
    cm = ref.ref_cmodel_build(L, E, K, dh, di, 7, 3, 16, 0.8, 2, 64, 4)
    assert cm, O.ref_error()
    floq = tmp_path / "m.floq"
    assert ref.ref_cmodel_save(cm, str(floq).encode()) == 0
    nt = 3
    toks = np.stack([O.token_input(1, t, dh) for t in range(nt)]).astype(np.float32)
    toks.tofile(tmp_path / "tokens.f32")
    out = tmp_path / "out"
    out.mkdir()
    exe = build(tmp_path)
    r = subprocess.run([str(exe), str(floq), str(tmp_path / "tokens.f32"), str(nt), str(out)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr + r.stdout
    got_u = np.fromfile(out / "u.f32", np.float32).reshape(nt * L, dh)
    got_sel = np.fromfile(out / "sel.u32", np.uint32).reshape(nt * L, K)
    got_w = np.fromfile(out / "w.f32", np.float32).reshape(nt * L, K)
    got_m = np.fromfile(out / "masks.u8", np.uint8).reshape(nt * L, K, di)
    got_y = np.fromfile(out / "y.f32", np.float32).reshape(nt * L, dh)
    got_y2 = np.fromfile(out / "y_untraced.f32", np.float32).reshape(nt * L, dh)
    # traced == untraced (test_model.cpp:263-279) up to the order of the
    # cross-CTA fp32 reductions into y
    assert O.rel_l2(got_y, got_y2) <= 1e-6
    i = 0
    for t in range(nt):
        h = toks[t].copy()
        for layer in range(L):
            u = np.empty(dh, np.float32)
            sel = np.empty(K, np.uint32)
            w = np.empty(K, np.float32)
            masks = np.empty((K, di), np.uint8)
            y = np.empty(dh, np.float32)
            assert ref.ref_layer_forward_traced(cm, layer, h, u, sel, w, masks, y) == 0
            assert O.rel_l2(got_u[i], u) <= 1e-5
            assert np.array_equal(got_sel[i], sel)
            assert np.allclose(got_w[i], w, rtol=1e-5, atol=1e-6)
            # masks: identical except ties (|v| within 1e-3 of the threshold)
            for j in range(K):
                diff = np.nonzero(got_m[i][j] != masks[j])[0]
                if len(diff):
                    eh = ref.ref_cmodel_expert(cm, layer, int(sel[j]))
                    v = _ref_qgemv(ref, eh, dh, di, u)
                    thr = _ref_threshold(ref, eh, dh, di)
                    assert np.all(np.abs(np.abs(v[diff]) - thr) <= 1e-3)
            assert O.rel_l2(got_y[i], y) <= 1e-2
            h = got_y[i].copy()  # chain on our output, like cmd_run
            i += 1
    # expert_forward_sparse / qgemv_channels on layer 0 expert 0
    ex = ref.ref_cmodel_expert(cm, 0, 0)
    x = toks[0].copy()
    y = np.empty(dh, np.float32)
    assert ref.ref_expert_forward(ex, x, y) == 0
    assert O.rel_l2(np.fromfile(out / "expert_y.f32", np.float32), y) <= 1e-2
    # qgemv_channels on layer 0 expert 0, predict_mask on layer 1 expert 0
    v = _ref_qgemv(ref, ex, dh, di, x)
    assert np.all(np.abs(np.fromfile(out / "qgemv_v.f32", np.float32) - v) <=
                  2e-5 + 2e-5 * np.abs(v))
    ex1 = ref.ref_cmodel_expert(cm, 1, 0)
    v1 = _ref_qgemv(ref, ex1, dh, di, x)
    t1 = _ref_threshold(ref, ex1, dh, di)
    m1 = np.fromfile(out / "predict_mask.u8", np.uint8)
    diff = np.nonzero(m1 != (np.abs(v1) >= t1))[0]
    assert np.all(np.abs(np.abs(v1[diff]) - t1) <= 1e-3)
    # predict_experts with the layer-0 router as the map (bias 0)
    rp = ct.POINTER(ct.c_float)()
    mp = ct.POINTER(ct.c_float)()
    ref.ref_cmodel_layer_view(cm, 0, ct.byref(rp), ct.byref(mp))
    router = np.ctypeslib.as_array(rp, shape=(E * dh,)).reshape(E, dh).copy()
    want = O.predict_experts(router, np.zeros(E, np.float32), x, K)
    assert np.array_equal(np.fromfile(out / "predict_experts.u32", np.uint32), want)
    ref.ref_cmodel_destroy(cm)


INTEG = ROOT / "tests" / "cpp" / "build" / "test_integration"


def test_integration_binary_built():
    """INTEGRATION.md's binding compiled with the reference's own headers and
    sources (tests/cpp/Makefile; built by `make` / build() where the reference
    exists, shipped prebuilt otherwise)."""
    if not INTEG.exists():
        if Path("/root/reference/proj/core/src").exists():
            subprocess.run(["make", "-C", str(ROOT / "tests" / "cpp")], check=True,
                           capture_output=True)
        else:
            pytest.skip("reference sources absent and no prebuilt test_integration")
    assert INTEG.exists()


@pytest.mark.gpu
def test_integration_reference_types_two_threads():
    """floe::gpu:: on the reference's own CompressedModel objects, 1 and 2 host
    threads: equal outputs, reference parity, the reference's error messages."""
    if not INTEG.exists():
        pytest.skip("tests/cpp/build/test_integration not built")
    r = subprocess.run([str(INTEG)], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:] + r.stdout[-1000:]
    assert "0 failures" in r.stdout
