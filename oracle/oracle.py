"""ctypes/numpy front end for the CPU checkers.

TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs -- never by the product
package (paper_2505_05950_b200), which must fail loudly without its CUDA
library instead of falling back here.

Two libraries:
  * ``C``   -- oracle/liboracle.so, the plain-C restatement (floe_oracle.c);
  * ``REF`` -- oracle/_ref/libfloe_ref.so, the unmodified reference core
               compiled from /root/reference/proj/core/src (None if absent).
"""
from __future__ import annotations

import ctypes as ct
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
THREADS = max(1, min(64, os.cpu_count() or 1))

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_sz, _u32, _u64, _int, _flt, _dbl, _vp = (ct.c_size_t, ct.c_uint32, ct.c_uint64,
                                          ct.c_int, ct.c_float, ct.c_double, ct.c_void_p)


def _sig(lib, name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


def _load_c():
    path = HERE / "liboracle.so"
    if not path.exists():
        raise RuntimeError(f"{path} missing: run `make -C oracle` (or __graft_entry__.build())")
    lib = ct.CDLL(str(path))
    _sig(lib, "fo_normals", None, _u64, _u64, _flt, _sz, _f32p, _int)
    _sig(lib, "fo_fill_gaussian", None, _f32p, _sz, _u64, _u64, _flt, _int)
    _sig(lib, "fo_weight_stream", _u64, _u64, _u64, _u64)
    _sig(lib, "fo_token_input", None, _u64, _u64, _u32, _f32p)
    _sig(lib, "fo_f32_to_f16_array", None, _f32p, _sz, _u16p, _int)
    _sig(lib, "fo_f16_to_f32_array", None, _u16p, _sz, _f32p)
    _sig(lib, "fo_packed_code_bytes", _sz, _sz, ct.c_uint)
    _sig(lib, "fo_quantize", _int, _f32p, _sz, ct.c_uint, _u32, _u8p, _u16p, _u16p, _int)
    _sig(lib, "fo_dequantize", _int, _u8p, _u16p, _u16p, _sz, ct.c_uint, _u32, _f32p, _int)
    _sig(lib, "fo_qgemv_channels", _int, _u8p, _u16p, _u16p, _sz, ct.c_uint, _u32, _sz,
         _f32p, _f32p, _int)
    _sig(lib, "fo_compression_ratio", _dbl, _sz, _sz, ct.c_uint, _u32, _dbl, _int)
    _sig(lib, "fo_gemv", None, _sz, _sz, _f32p, _f32p, _f32p)
    _sig(lib, "fo_silu", _flt, _flt)
    _sig(lib, "fo_softmax_inplace", None, _f32p, _sz)
    _sig(lib, "fo_top_k", _int, _f32p, _sz, _sz, _u32p)
    _sig(lib, "fo_calibrate_threshold", _flt, _f32p, _sz, _dbl)
    _sig(lib, "fo_sparsity_mask", None, _f32p, _sz, _flt, _u8p)
    _sig(lib, "fo_expert_forward_sparse", None, _u32, _u32, ct.c_uint, _u32, _u8p, _u16p,
         _u16p, _f32p, _f32p, _flt, _f32p, _f32p, _vp, _vp, _int)
    _sig(lib, "fo_expert_forward_dense", None, _u32, _u32, _f32p, _f32p, _f32p, _f32p, _f32p)
    _sig(lib, "fo_route", _int, _f32p, _u32, _u32, _f32p, _u32, _u32p, _f32p)
    _sig(lib, "fo_predict_mask", _int, _u8p, _u16p, _u16p, _sz, ct.c_uint, _u32, _u32,
         _f32p, _flt, _u8p, _int)
    _sig(lib, "fo_predict_experts", _int, _f32p, _f32p, _u32, _u32, _f32p, _u32, _u32p)
    _sig(lib, "fo_pack_compact", ct.c_long, _u32, _u32, _f32p, _f32p, _u8p, _u32, _u32p, _u8p)
    return lib


def _load_ref():
    path = HERE / "_ref" / "libfloe_ref.so"
    if not path.exists():
        return None
    lib = ct.CDLL(str(path))
    _sig(lib, "ref_last_error", ct.c_char_p)
    _sig(lib, "ref_normals", None, _u64, _u64, _sz, _f32p)
    _sig(lib, "ref_uniforms", None, _u64, _u64, _sz, _f64p)
    _sig(lib, "ref_seeded_expert", None, _u32, _u32, _u64, _f32p, _f32p, _f32p)
    _sig(lib, "ref_token_input", None, _u64, _u64, _u32, _f32p)
    _sig(lib, "ref_f32_to_f16", None, _f32p, _sz, _u16p)
    _sig(lib, "ref_f16_to_f32", None, _u16p, _sz, _f32p)
    _sig(lib, "ref_packed_code_bytes", _sz, _sz, ct.c_uint)
    _sig(lib, "ref_quantize", _int, _f32p, _sz, ct.c_uint, _u32, _u8p, _u16p, _u16p)
    _sig(lib, "ref_dequantize", _int, _u8p, _u16p, _u16p, _sz, ct.c_uint, _u32, _f32p)
    _sig(lib, "ref_qgemv_channels", _int, _u8p, _u16p, _u16p, _sz, ct.c_uint, _u32, _sz,
         _f32p, _f32p)
    _sig(lib, "ref_compression_ratio", _dbl, _sz, _sz, ct.c_uint, _u32, _dbl, _int)
    _sig(lib, "ref_top_k", _int, _f32p, _sz, _sz, _u32p)
    _sig(lib, "ref_softmax", None, _f32p, _sz)
    _sig(lib, "ref_silu", _flt, _flt)
    _sig(lib, "ref_calibrate_threshold", _flt, _f32p, _sz, _dbl)
    _sig(lib, "ref_route", _int, _f32p, _u32, _u32, _f32p, _u32, _u32p, _f32p)
    _sig(lib, "ref_expert_create", _vp, _u32, _u32, ct.c_uint, _u32, _u8p, _u16p, _u16p,
         _f32p, _f32p, _flt)
    _sig(lib, "ref_expert_compress", _vp, _u32, _u32, _f32p, _f32p, _f32p, ct.c_uint, _u32,
         _flt)
    _sig(lib, "ref_expert_destroy", None, _vp)
    _sig(lib, "ref_expert_set_threshold", None, _vp, _flt)
    _sig(lib, "ref_expert_view", None, _vp, ct.POINTER(ct.POINTER(ct.c_uint8)),
         ct.POINTER(ct.POINTER(ct.c_uint16)), ct.POINTER(ct.POINTER(ct.c_uint16)),
         ct.POINTER(ct.POINTER(ct.c_float)), ct.POINTER(ct.POINTER(ct.c_float)),
         ct.POINTER(ct.c_float))
    _sig(lib, "ref_expert_forward", _int, _vp, _f32p, _f32p)
    _sig(lib, "ref_expert_forward_replicas", _dbl, _vp, _f32p, ct.c_uint, ct.c_uint)
    _sig(lib, "ref_expert_forward_dense", _int, _u32, _u32, _f32p, _f32p, _f32p, _f32p, _f32p)
    _sig(lib, "ref_pack_compact", _int, _vp, _u8p, _u32, _u32p, _u8p, ct.POINTER(ct.c_uint64))
    _sig(lib, "ref_predict_mask", _int, _u8p, _u16p, _u16p, _sz, ct.c_uint, _u32, _u32,
         _f32p, _flt, _u8p)
    _sig(lib, "ref_predict_experts", _int, _f32p, _f32p, _u32, _u32, _f32p, _u32, _u32p)
    _sig(lib, "ref_cmodel_build", _vp, _u32, _u32, _u32, _u32, _u32, _u64, _u64, _u64, _dbl,
         ct.c_uint, _u32, ct.c_uint)
    _sig(lib, "ref_cmodel_build_thresholds", _vp, _u32, _u32, _u32, _u32, _u32, _u64, _f32p,
         ct.c_uint, _u32, ct.c_uint)
    _sig(lib, "ref_layer_forward_replicas", _dbl, _vp, _u32, _f32p, _u32, ct.c_uint)
    _sig(lib, "ref_layer_calls_replicas", _dbl, _vp, _u32, _f32p, _u32, ct.c_uint)
    _sig(lib, "ref_cmodel_build_replay", _vp, _u32, _u32, _u32, _u32, _u32, _u64, _u64, _u64,
         _dbl, ct.c_uint, _u32, ct.c_uint, _f32p)
    _sig(lib, "ref_calibrate_weights", _int, _u32, _u32, _u32, _u32, _u32, _f32p, _f32p, _f32p,
         _f32p, _f32p, _u64, _u64, _dbl, _u64, ct.c_uint, _flt, _f32p)
    _sig(lib, "ref_cmodel_load", _vp, ct.c_char_p)
    _sig(lib, "ref_cmodel_save", _int, _vp, ct.c_char_p)
    _sig(lib, "ref_cmodel_destroy", None, _vp)
    _sig(lib, "ref_cmodel_dims", None, _vp, _u32p, ct.POINTER(ct.c_uint), ct.POINTER(ct.c_uint32))
    _sig(lib, "ref_cmodel_layer_view", None, _vp, _u32, ct.POINTER(ct.POINTER(ct.c_float)),
         ct.POINTER(ct.POINTER(ct.c_float)))
    _sig(lib, "ref_cmodel_expert", _vp, _vp, _u32, _u32)
    _sig(lib, "ref_layer_forward", _int, _vp, _u32, _f32p, _f32p)
    _sig(lib, "ref_layer_forward_traced", _int, _vp, _u32, _f32p, _f32p, _u32p, _f32p, _u8p,
         _f32p)
    return lib


C = _load_c()
REF = _load_ref()


def ref_error() -> str:
    return REF.ref_last_error().decode() if REF is not None else "reference library absent"


# --------------------------------------------------------------------------
# numpy helpers over the C restatement

def normals(seed: int, stream: int, n: int, scale: float = 1.0) -> np.ndarray:
    out = np.empty(n, np.float32)
    C.fo_normals(seed, stream, np.float32(scale), n, out, THREADS)
    return out


def seeded_expert(dh: int, di: int, seed: int):
    """acceptance_test.cpp:38-53: gate/up/down on Rng(seed, 1/2/3) x 1/sqrt(dh)."""
    sd = np.float32(1.0) / np.sqrt(np.float32(dh), dtype=np.float32)
    n = dh * di
    return tuple(normals(seed, s, n, float(sd)) for s in (1, 2, 3))


def seeded_input(dh: int, seed: int, stream: int = 4) -> np.ndarray:
    """acceptance_test.cpp:55-60 (stream 4); test_model.cpp:45-49 uses stream 9."""
    return normals(seed, stream, dh, 1.0)


def token_input(seed: int, t: int, dh: int) -> np.ndarray:
    out = np.empty(dh, np.float32)
    C.fo_token_input(seed, t, dh, out)
    return out


def f32_to_f16(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32).ravel()
    out = np.empty(x.size, np.uint16)
    C.fo_f32_to_f16_array(x, x.size, out, THREADS)
    return out


def f16_to_f32(h: np.ndarray) -> np.ndarray:
    h = np.ascontiguousarray(h, np.uint16).ravel()
    out = np.empty(h.size, np.float32)
    C.fo_f16_to_f32_array(h, h.size, out)
    return out


def fp16_round(x: np.ndarray) -> np.ndarray:
    """f32 -> f16 (reference RNE) -> f32: the values a fp16 record carries."""
    return f16_to_f32(f32_to_f16(x)).reshape(np.shape(x))


class Quantized:
    """Mirror of floe::QuantizedTensor (core/include/floe/quant.hpp:20-31)."""

    def __init__(self, codes, scales, zeros, n, bits, group_size):
        self.codes, self.scales, self.zeros = codes, scales, zeros
        self.n, self.bits, self.group_size = n, bits, group_size

    def stored_bytes(self, include_metadata=True):
        return self.codes.size + (2 * self.scales.size + 2 * self.zeros.size
                                  if include_metadata else 0)


def quantize(x: np.ndarray, bits: int, group_size: int) -> Quantized:
    x = np.ascontiguousarray(x, np.float32).ravel()
    n = x.size
    nb = C.fo_packed_code_bytes(n, bits)
    ng = n // group_size if group_size else 0
    codes = np.zeros(nb, np.uint8)
    scales = np.zeros(max(ng, 1), np.uint16)
    zeros = np.zeros(max(ng, 1), np.uint16)
    rc = C.fo_quantize(x, n, bits, group_size, codes, scales, zeros, THREADS)
    if rc != 0:
        raise ValueError({-1: "quantize: bits must be one of {1,2,3,4,8}",
                          -2: "quantize: group_size must divide element count",
                          -3: "quantize: non-finite input"}[rc])
    return Quantized(codes, scales[:ng], zeros[:ng], n, bits, group_size)


def dequantize(q: Quantized) -> np.ndarray:
    out = np.empty(q.n, np.float32)
    if C.fo_dequantize(q.codes, q.scales, q.zeros, q.n, q.bits, q.group_size, out,
                       THREADS) != 0:
        raise ValueError("quantized tensor: corrupt packing")
    return out


def qgemv_channels(q: Quantized, ch_len: int, x: np.ndarray) -> np.ndarray:
    y = np.empty(q.n // ch_len, np.float32)
    if C.fo_qgemv_channels(q.codes, q.scales, q.zeros, q.n, q.bits, q.group_size, ch_len,
                           np.ascontiguousarray(x, np.float32), y, THREADS) != 0:
        raise ValueError("qgemv_channels: ch_len must divide element count")
    return y


def sparsity_mask(v: np.ndarray, t: float) -> np.ndarray:
    v = np.ascontiguousarray(v, np.float32)
    m = np.empty(v.size, np.uint8)
    C.fo_sparsity_mask(v, v.size, np.float32(t), m)
    return m


def calibrate_threshold(mags: np.ndarray, k: float) -> float:
    m = np.array(mags, np.float32, copy=True)
    return float(C.fo_calibrate_threshold(m, m.size, k))


class Expert:
    """Mirror of floe::CompressedExpert (core/include/floe/model.hpp:60-70)."""

    def __init__(self, dh, di, up_q: Quantized, gate, down_t, threshold):
        self.d_hidden, self.d_intermediate = dh, di
        self.up_q = up_q
        self.gate = np.ascontiguousarray(gate, np.float32).ravel()
        self.down_t = np.ascontiguousarray(down_t, np.float32).ravel()
        self.threshold = float(threshold)


def compress_expert(dh, di, gate, up, down, bits, group_size, threshold) -> Expert:
    return Expert(dh, di, quantize(up, bits, group_size), gate, down, threshold)


def expert_forward_sparse(e: Expert, x: np.ndarray, want_v=False):
    y = np.empty(e.d_hidden, np.float32)
    v = np.empty(e.d_intermediate, np.float32)
    mask = np.empty(e.d_intermediate, np.uint8)
    q = e.up_q
    C.fo_expert_forward_sparse(e.d_hidden, e.d_intermediate, q.bits, q.group_size, q.codes,
                               q.scales, q.zeros, e.gate, e.down_t, np.float32(e.threshold),
                               np.ascontiguousarray(x, np.float32), y,
                               v.ctypes.data, mask.ctypes.data, THREADS)
    return (y, v, mask) if want_v else y


def expert_forward_dense(dh, di, gate, up, down, x):
    y = np.empty(dh, np.float32)
    C.fo_expert_forward_dense(dh, di, gate, up, down, np.ascontiguousarray(x, np.float32), y)
    return y


def top_k(v: np.ndarray, k: int) -> np.ndarray:
    v = np.ascontiguousarray(v, np.float32)
    out = np.empty(k, np.uint32)
    if C.fo_top_k(v, v.size, k, out) != 0:
        raise ValueError("top_k: k out of range")
    return out


def route(router: np.ndarray, u: np.ndarray, k: int):
    E, dh = router.shape
    sel = np.empty(k, np.uint32)
    w = np.empty(k, np.float32)
    if C.fo_route(np.ascontiguousarray(router, np.float32), E, dh,
                  np.ascontiguousarray(u, np.float32), k, sel, w) != 0:
        raise ValueError("top_k: k out of range")
    return sel, w


def predict_mask(q: Quantized, dh: int, x_prev: np.ndarray, t: float) -> np.ndarray:
    mask = np.empty(q.n // dh, np.uint8)
    if C.fo_predict_mask(q.codes, q.scales, q.zeros, q.n, q.bits, q.group_size, dh,
                         np.ascontiguousarray(x_prev, np.float32), np.float32(t), mask,
                         THREADS) != 0:
        raise ValueError("predict_mask: tensor not channel-divisible")
    return mask


def predict_experts(w: np.ndarray, b: np.ndarray, x: np.ndarray, count: int) -> np.ndarray:
    E, dh = w.shape
    out = np.empty(count, np.uint32)
    if C.fo_predict_experts(np.ascontiguousarray(w, np.float32),
                            np.ascontiguousarray(b, np.float32), E, dh,
                            np.ascontiguousarray(x, np.float32), count, out) != 0:
        raise ValueError("top_k: k out of range")
    return out


def pack_compact(e: Expert, mask: np.ndarray, element_bytes: int):
    di, dh = e.d_intermediate, e.d_hidden
    mask = np.ascontiguousarray(mask, np.uint8)
    n = int(mask.astype(bool).sum())
    ch = np.empty(max(n, 1), np.uint32)
    payload = np.empty(max(n, 1) * 2 * dh * element_bytes, np.uint8)
    got = C.fo_pack_compact(dh, di, e.gate, e.down_t, mask, element_bytes, ch, payload)
    if got < 0:
        raise ValueError("pack_compact: element_bytes must be 2 or 4")
    return ch[:got], payload[: got * 2 * dh * element_bytes]


class Layer:
    """One compressed MoE block: router [E][dh], mixing [dh][dh], experts."""

    def __init__(self, router, mixing, experts, top_k):
        self.router = np.ascontiguousarray(router, np.float32)
        self.mixing = np.ascontiguousarray(mixing, np.float32)
        self.experts = experts
        self.top_k = top_k


class _FoLayer(ct.Structure):
    _fields_ = [("d_hidden", ct.c_uint32), ("d_intermediate", ct.c_uint32),
                ("n_experts", ct.c_uint32), ("top_k", ct.c_uint32), ("bits", ct.c_uint),
                ("group_size", ct.c_uint32), ("router", ct.c_void_p), ("mixing", ct.c_void_p),
                ("codes", ct.c_void_p), ("scales", ct.c_void_p), ("zeros", ct.c_void_p),
                ("gate", ct.c_void_p), ("down_t", ct.c_void_p), ("thresholds", ct.c_void_p)]


def layer_forward(L: Layer, h: np.ndarray, traced=False):
    """block_forward / layer_forward(CompressedModel) (model.cpp:145-190)."""
    E = len(L.experts)
    e0 = L.experts[0]
    dh, di = e0.d_hidden, e0.d_intermediate
    arr = lambda xs: (ct.c_void_p * E)(*[a.ctypes.data for a in xs])
    keep = [arr([e.up_q.codes for e in L.experts]), arr([e.up_q.scales for e in L.experts]),
            arr([e.up_q.zeros for e in L.experts]), arr([e.gate for e in L.experts]),
            arr([e.down_t for e in L.experts])]
    th = np.array([e.threshold for e in L.experts], np.float32)
    s = _FoLayer(dh, di, E, L.top_k, e0.up_q.bits, e0.up_q.group_size, L.router.ctypes.data,
                 L.mixing.ctypes.data, ct.addressof(keep[0]), ct.addressof(keep[1]),
                 ct.addressof(keep[2]), ct.addressof(keep[3]), ct.addressof(keep[4]),
                 th.ctypes.data)
    fn = C.fo_layer_forward
    fn.restype = ct.c_int
    fn.argtypes = [ct.POINTER(_FoLayer), ct.c_void_p, ct.c_void_p, ct.c_void_p, ct.c_void_p,
                   ct.c_void_p, ct.c_void_p, ct.c_int]
    h = np.ascontiguousarray(h, np.float32)
    y = np.empty(dh, np.float32)
    u = np.empty(dh, np.float32)
    sel = np.empty(L.top_k, np.uint32)
    w = np.empty(L.top_k, np.float32)
    masks = np.empty((L.top_k, di), np.uint8)
    rc = fn(ct.byref(s), h.ctypes.data, y.ctypes.data, u.ctypes.data, sel.ctypes.data,
            w.ctypes.data, masks.ctypes.data, THREADS)
    if rc != 0:
        raise ValueError("layer_forward failed")
    if traced:
        return dict(block_input=u, experts=sel, weights=w, masks=masks, out=y)
    return y


def rel_l2(got, ref) -> float:
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    return float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30))
