"""ctypes binding of include/floe_gpu.h (the product's C ABI).

Device memory and streams come from PyTorch (plumbing only): device inputs are
``torch.Tensor``s on ``cuda``, and ``stream`` defaults to torch's current
stream so calls compose with torch ordering and CUDA-graph capture.
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "libfloe_b200.so"
if os.environ.get("FLOE_LIB"):  # A/B builds of the same ABI (tools/, never the default)
    _LIB_PATH = Path(os.environ["FLOE_LIB"]).resolve()

FLOE_OK = 0
_STATUS = {1: "FLOE_ERR_INVALID", 2: "FLOE_ERR_CUDA", 3: "FLOE_ERR_OOM", 4: "FLOE_ERR_UNSUPPORTED"}


class FloeError(RuntimeError):
    """A nonzero floe_status; the message keeps the reference's '<fn>: <reason>' form."""

    def __init__(self, msg: str, status: int = 1):
        super().__init__(msg)
        self.status = status


class ExpertHostView(ct.Structure):
    _fields_ = [("d_hidden", ct.c_uint32), ("d_intermediate", ct.c_uint32),
                ("bits", ct.c_uint32), ("group_size", ct.c_uint32),
                ("codes", ct.c_void_p), ("scales", ct.c_void_p), ("zeros", ct.c_void_p),
                ("gate_f32", ct.c_void_p), ("down_f32", ct.c_void_p),
                ("records_f16", ct.c_void_p), ("threshold", ct.c_float),
                ("flags", ct.c_uint32)]


FLOE_VIEW_DEVICE = 1
FLOE_VIEW_HOST_RECORDS = 2


class ExpertInfo(ct.Structure):
    _fields_ = [("d_hidden", ct.c_uint32), ("d_intermediate", ct.c_uint32),
                ("bits", ct.c_uint32), ("group_size", ct.c_uint32), ("threshold", ct.c_float),
                ("code_bytes", ct.c_uint64), ("meta_bytes", ct.c_uint64),
                ("record_bytes", ct.c_uint64), ("fast_path", ct.c_int)]


class LayerHostView(ct.Structure):
    _fields_ = [("d_hidden", ct.c_uint32), ("n_experts", ct.c_uint32), ("top_k", ct.c_uint32),
                ("router", ct.c_void_p), ("mixing", ct.c_void_p), ("mixing_f16", ct.c_int),
                ("experts", ct.c_void_p)]


class LayerTrace(ct.Structure):
    _fields_ = [("block_input_dev", ct.c_void_p), ("experts_dev", ct.c_void_p),
                ("weights_dev", ct.c_void_p), ("masks_dev", ct.c_void_p)]


class FloatLayerView(ct.Structure):
    _fields_ = [("router", ct.c_void_p), ("mixing", ct.c_void_p), ("gate", ct.c_void_p),
                ("up", ct.c_void_p), ("down_t", ct.c_void_p)]


_P = ct.c_void_p
_U32 = ct.c_uint32
_F = ct.c_float
# name -> (restype, argtypes); the full exported surface of include/floe_gpu.h
_SIGS = {
    "floe_gpu_last_error": (ct.c_char_p, []),
    "floe_gpu_abi_version": (ct.c_int, []),
    "floe_gpu_device_malloc": (ct.c_int, [_P, ct.c_size_t]),
    "floe_gpu_offload_create": (ct.c_int, [_P, _U32, ct.c_uint64, _P]),
    "floe_gpu_offload_destroy": (ct.c_int, [_P]),
    "floe_gpu_offload_decode": (ct.c_int, [_P, _P, _P, _P, _P]),
    "floe_gpu_offload_decode_replay": (ct.c_int, [_P, _P, _P, _P, _P]),
    "floe_gpu_offload_stats": (ct.c_int, [_P, _P, _P]),
    "floe_gpu_offload_set_eval": (ct.c_int, [_P, ct.c_int, _P, _U32]),
    "floe_gpu_expert_download": (ct.c_int, [_P, _P, _P, _P, _P]),
    "floe_gpu_record_cache_save": (ct.c_int, [_P, _U32, ct.c_char_p]),
    "floe_gpu_record_cache_info": (ct.c_int, [ct.c_char_p, _P]),
    "floe_gpu_record_cache_load": (ct.c_int, [ct.c_char_p, _U32, _P, _P]),
    "floe_gpu_expert_set_resident": (ct.c_int, [_P, ct.c_int, _P]),
    "floe_gpu_expert_residency": (ct.c_int, [_P, _P, _P]),
    "floe_gpu_device_free": (ct.c_int, [_P]),
    "floe_gpu_copy": (ct.c_int, [_P, _P, ct.c_size_t, _P]),
    "floe_gpu_device_info": (ct.c_int, [_P, _P, _P, _P]),
    "floe_gpu_expert_create": (ct.c_int, [ct.POINTER(ExpertHostView), ct.POINTER(_P)]),
    "floe_gpu_expert_destroy": (ct.c_int, [_P]),
    "floe_gpu_expert_info": (ct.c_int, [_P, ct.POINTER(ExpertInfo)]),
    "floe_gpu_expert_set_threshold": (ct.c_int, [_P, _F]),
    "floe_gpu_workspace_create": (ct.c_int, [_U32, _U32, _U32, ct.POINTER(_P)]),
    "floe_gpu_workspace_destroy": (ct.c_int, [_P]),
    "floe_gpu_expert_forward_sparse": (ct.c_int, [_P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "floe_gpu_expert_forward_sparse_host": (ct.c_int, [_P, _P, _P, _P, _P, _P, _P]),
    "floe_gpu_qgemv_channels": (ct.c_int, [_P, _P, _P, _P, _P]),
    "floe_gpu_qgemv_channels_batched": (ct.c_int, [_P, _P, ct.c_uint32, _P, _P]),
    "floe_gpu_expert_forward_batched": (ct.c_int, [_P, _P, ct.c_uint32, _P, _P, _P]),
    "floe_gpu_expert_forward_prefill": (ct.c_int, [_P, _P, ct.c_uint32, _P, _P]),
    "floe_gpu_dequantize_up": (ct.c_int, [_P, _P, _P]),
    "floe_gpu_predict_mask": (ct.c_int, [_P, _P, _P, _F, _P, _P, _P, _P]),
    "floe_gpu_layer_create": (ct.c_int, [ct.POINTER(LayerHostView), ct.POINTER(_P)]),
    "floe_gpu_layer_destroy": (ct.c_int, [_P]),
    "floe_gpu_layer_forward": (ct.c_int, [_P, _P, _P, _P, ct.POINTER(LayerTrace), _P]),
    "floe_gpu_layer_forward_host": (ct.c_int, [_P, _P, _P, _P, _P]),
    "floe_gpu_workspace_reset_counters": (ct.c_int, [_P, _P]),
    "floe_gpu_workspace_read_counters": (ct.c_int, [_P, _P, _P, _P]),
    "floe_gpu_workspace_set_profiling": (ct.c_int, [_P, ct.c_int]),
    "floe_gpu_workspace_read_profile": (ct.c_int, [_P, _P, _P]),
    "floe_gpu_workspace_set_phase_trace": (ct.c_int, [_P, ct.c_int]),
    "floe_gpu_workspace_read_phase_trace": (ct.c_int, [_P, _P, _U32, _P]),
    "floe_gpu_gen_normals":(ct.c_int, [ct.c_uint64, ct.c_uint64, ct.c_uint64, _F, ct.c_int, _P,
                                        _P]),
    "floe_gpu_quantize": (ct.c_int, [_P, ct.c_uint64, _U32, _U32, _P, _P, _P, _P]),
    "floe_gpu_predictor_create": (ct.c_int, [_U32, _U32, _U32, _P, _P, ct.POINTER(_P)]),
    "floe_gpu_predictor_destroy": (ct.c_int, [_P]),
    "floe_gpu_predict_experts": (ct.c_int, [_P, _P, _U32, _U32, _P, _P]),
    "floe_gpu_pack_compact": (ct.c_int, [_P, _P, _U32, _P, _P, _P, _P]),
    "floe_gpu_layer_forward_batched": (ct.c_int, [_P, _P, _P, _U32, _P, _P]),
    "floe_gpu_model_create": (ct.c_int, [_P, _U32, ct.POINTER(_P)]),
    "floe_gpu_model_destroy": (ct.c_int, [_P]),
    "floe_gpu_model_multi_layer": (ct.c_int, [_P]),
    "floe_gpu_model_decode": (ct.c_int, [_P, _P, _P, _P, ct.c_int, _P]),
    "floe_gpu_model_decode_host": (ct.c_int, [_P, _P, _P, _P, ct.c_int, _P]),
    "floe_gpu_calib_create": (ct.c_int, [_U32, _U32, _U32, _U32, ct.c_uint64, ct.c_uint64,
                                         ct.POINTER(_P)]),
    "floe_gpu_calib_destroy": (ct.c_int, [_P]),
    "floe_gpu_calib_layer": (ct.c_int, [_P, _U32, ct.POINTER(FloatLayerView), _U32, _F, _P, _P,
                                        _U32, _P]),
    "floe_gpu_calib_thresholds": (ct.c_int, [_P, ct.c_double, _P]),
}

_lib = None


def library_path() -> Path:
    return _LIB_PATH


def lib():
    """Load libfloe_b200.so (raises FloeError if it was never built)."""
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise FloeError(f"{_LIB_PATH} is not built: run `make` or __graft_entry__.build()", 2)
        L = ct.CDLL(str(_LIB_PATH))
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def exported_symbols() -> list[str]:
    """Dynamic symbols of the built library whose name starts with floe_gpu_."""
    out = subprocess.run(["nm", "-D", "--defined-only", str(_LIB_PATH)], check=True,
                         capture_output=True, text=True).stdout
    return sorted(l.split()[-1] for l in out.splitlines() if l.split()[-1].startswith("floe_gpu_"))


def _check(rc: int):
    if rc != FLOE_OK:
        raise FloeError(lib().floe_gpu_last_error().decode(), rc)


def abi_version() -> int:
    return lib().floe_gpu_abi_version()


def device_info() -> dict:
    sm, ma, mi, mem = ct.c_int(), ct.c_int(), ct.c_int(), ct.c_size_t()
    _check(lib().floe_gpu_device_info(ct.byref(sm), ct.byref(ma), ct.byref(mi), ct.byref(mem)))
    return dict(sm_count=sm.value, cc=(ma.value, mi.value), total_mem=mem.value)


# ---------------------------------------------------------------------------
def _torch():
    import torch
    return torch


def _ptr(t) -> int:
    if t is None:
        return 0
    if isinstance(t, int):
        return t
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def _stream(stream) -> int:
    if stream is None:
        torch = _torch()
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _dev_f32(x, n: int, fn: str):
    torch = _torch()
    if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float32):
        raise FloeError(f"{fn}: expected a float32 CUDA tensor")
    if x.numel() != n:
        raise FloeError(f"{fn}: dimension mismatch")
    return x.contiguous()


class Workspace:
    """Per-stream scratch (floe_gpu_workspace)."""

    def __init__(self, d_hidden: int, d_intermediate: int, max_slots: int = 1):
        h = ct.c_void_p()
        _check(lib().floe_gpu_workspace_create(d_hidden, d_intermediate, max_slots, ct.byref(h)))
        self.handle = h.value
        self.d_hidden, self.d_intermediate, self.max_slots = d_hidden, d_intermediate, max_slots

    def close(self):
        if getattr(self, "handle", None):
            lib().floe_gpu_workspace_destroy(self.handle)
            self.handle = None

    __del__ = close

    STAGES = ("mixing", "route", "k1_up_threshold", "k2_gate_down", "fused")

    def reset_counters(self, stream=None):
        _check(lib().floe_gpu_workspace_reset_counters(self.handle, _stream(stream)))

    def read_counters(self, stream=None) -> dict:
        calls, kept = ct.c_uint64(), ct.c_uint64()
        _check(lib().floe_gpu_workspace_read_counters(self.handle, ct.byref(calls),
                                                      ct.byref(kept), _stream(stream)))
        return dict(calls=calls.value, kept=kept.value)

    def set_profiling(self, enable: bool):
        _check(lib().floe_gpu_workspace_set_profiling(self.handle, 1 if enable else 0))

    def set_phase_trace(self, enable: bool):
        _check(lib().floe_gpu_workspace_set_phase_trace(self.handle, 1 if enable else 0))

    def read_phase_trace(self) -> np.ndarray:
        """[grid, 8] %globaltimer ns marks of the fused kernel's last call."""
        out = np.zeros(96 * 1024, np.uint64)
        grid = ct.c_uint32()
        _check(lib().floe_gpu_workspace_read_phase_trace(self.handle, out.ctypes.data, out.size,
                                                         ct.byref(grid)))
        return out[: 96 * grid.value].reshape(grid.value, 96)

    def read_profile(self) -> dict:
        ms = (ct.c_double * 5)()
        n = (ct.c_uint64 * 5)()
        _check(lib().floe_gpu_workspace_read_profile(self.handle, ms, n))
        return {k: dict(ms=ms[i], launches=n[i]) for i, k in enumerate(self.STAGES)}


class GpuExpert:
    """A compressed expert resident in HBM (floe::CompressedExpert on the device).

    codes/scales/zeros are the reference's QuantizedTensor arrays; gate/down are
    f32 [di][dh] (converted to f16 records on upload) or ``records`` is the
    pack_compact f16 wire format of all channels.
    """

    def __init__(self, d_hidden, d_intermediate, bits, group_size, codes, scales, zeros,
                 gate=None, down=None, records=None, threshold=0.0, host_records=False):
        keep = []
        on_device = not isinstance(codes, np.ndarray)  # torch CUDA tensors

        def host(a, dt):
            if a is None:
                return None
            if on_device:
                a = a.contiguous()
                keep.append(a)
                return a.data_ptr()
            a = np.ascontiguousarray(a, dt)
            keep.append(a)
            return a.ctypes.data

        v = ExpertHostView(d_hidden, d_intermediate, bits, group_size,
                           host(codes, np.uint8), host(scales, np.uint16), host(zeros, np.uint16),
                           host(gate, np.float32), host(down, np.float32),
                           host(records, np.uint16), float(threshold),
                           (FLOE_VIEW_DEVICE if on_device else 0)
                           | (FLOE_VIEW_HOST_RECORDS if host_records else 0))
        h = ct.c_void_p()
        _check(lib().floe_gpu_expert_create(ct.byref(v), ct.byref(h)))
        self.handle = h.value
        self.d_hidden, self.d_intermediate = d_hidden, d_intermediate
        self.bits, self.group_size = bits, group_size

    def close(self):
        if getattr(self, "handle", None):
            lib().floe_gpu_expert_destroy(self.handle)
            self.handle = None

    __del__ = close

    def info(self) -> dict:
        i = ExpertInfo()
        _check(lib().floe_gpu_expert_info(self.handle, ct.byref(i)))
        return {f: getattr(i, f) for f, _ in ExpertInfo._fields_}

    @property
    def threshold(self) -> float:
        return self.info()["threshold"]

    def set_resident(self, resident: bool, stream=None):
        """Move the gate|down records to HBM (True) or keep them host-resident
        (False; the kernels read them over PCIe).  Stream-ordered."""
        _check(lib().floe_gpu_expert_set_resident(self.handle, 1 if resident else 0,
                                                  _stream(stream)))

    def residency(self) -> dict:
        r, nb = ct.c_int(), ct.c_uint64()
        _check(lib().floe_gpu_expert_residency(self.handle, ct.byref(r), ct.byref(nb)))
        return dict(resident=bool(r.value), device_bytes=nb.value)

    def set_threshold(self, t: float):
        _check(lib().floe_gpu_expert_set_threshold(self.handle, float(t)))

    def download(self) -> dict:
        """The quantized up projection in the reference packing and the threshold."""
        n = self.d_hidden * self.d_intermediate
        codes = np.empty((n * self.bits + 7) // 8, np.uint8)
        scales = np.empty(n // self.group_size, np.uint16)
        zeros = np.empty_like(scales)
        t = ct.c_float()
        _check(lib().floe_gpu_expert_download(self.handle, codes.ctypes.data, scales.ctypes.data,
                                              zeros.ctypes.data, ct.byref(t)))
        return dict(codes=codes, scales=scales, zeros=zeros, threshold=t.value)

    @classmethod
    def _adopt(cls, handle, d_hidden, d_intermediate, bits, group_size):
        e = cls.__new__(cls)
        e.handle = handle
        e.d_hidden, e.d_intermediate = d_hidden, d_intermediate
        e.bits, e.group_size = bits, group_size
        return e

    def bytes_per_token(self, n_kept: int) -> int:
        """Algorithmic HBM bytes of one expert-token."""
        i = self.info()
        return (i["code_bytes"] + i["meta_bytes"] + n_kept * i["record_bytes"]
                + 8 * self.d_hidden)

    # -- raw device call (pointers as ints) ---------------------------------
    def forward_raw(self, ws: Workspace, x_ptr: int, y_ptr: int, v_ptr=0, mask_ptr=0,
                    kept_ptr=0, nkept_ptr=0, stream: int = 0):
        _check(lib().floe_gpu_expert_forward_sparse(self.handle, ws.handle, x_ptr, y_ptr,
                                                    v_ptr, mask_ptr, kept_ptr, nkept_ptr,
                                                    stream))


def expert_forward_sparse(e: GpuExpert, h, ws: Workspace, *, v=None, mask=None, kept=None,
                          n_kept=None, out=None, stream=None):
    """floe::expert_forward_sparse(const CompressedExpert&, const Vec&) (model.cpp:128-142).

    ``h`` on the device (torch CUDA tensor) -> stream-ordered device call; ``h``
    as a numpy array -> the host call (H2D, compute, D2H, synchronise).
    """
    if isinstance(h, np.ndarray):
        h = np.ascontiguousarray(h, np.float32)
        if h.size != e.d_hidden:
            raise FloeError("expert_forward_sparse: dimension mismatch")
        y = np.empty(e.d_hidden, np.float32) if out is None else out
        _check(lib().floe_gpu_expert_forward_sparse_host(
            e.handle, ws.handle, h.ctypes.data, y.ctypes.data, _ptr(v), _ptr(mask),
            _stream(stream) if stream is not None else 0))
        return y
    torch = _torch()
    h = _dev_f32(h, e.d_hidden, "expert_forward_sparse")
    y = torch.empty(e.d_hidden, dtype=torch.float32, device=h.device) if out is None else out
    e.forward_raw(ws, h.data_ptr(), y.data_ptr(), _ptr(v), _ptr(mask), _ptr(kept), _ptr(n_kept),
                  _stream(stream))
    return y


def qgemv_channels(e: GpuExpert, x, ws: Workspace, stream=None):
    """floe::qgemv_channels(up_q, d_hidden, x, y) (quant.cpp:122-136)."""
    torch = _torch()
    x = _dev_f32(x, e.d_hidden, "qgemv_channels")
    v = torch.empty(e.d_intermediate, dtype=torch.float32, device=x.device)
    _check(lib().floe_gpu_qgemv_channels(e.handle, ws.handle, x.data_ptr(), v.data_ptr(),
                                         _stream(stream)))
    return v


def qgemv_channels_batched(e: GpuExpert, x, stream=None):
    """qgemv_channels for a batch of tokens: x [B, d_hidden] -> v [B, d_intermediate]
    (tcgen05 tensor cores, exact integer group sums; B <= 64)."""
    torch = _torch()
    if x.dim() != 2 or x.shape[1] != e.d_hidden or x.dtype != torch.float32 or not x.is_cuda:
        raise FloeError("qgemv_channels_batched: x must be a cuda float32 [B, d_hidden]")
    x = x.contiguous()
    v = torch.empty((x.shape[0], e.d_intermediate), dtype=torch.float32, device=x.device)
    _check(lib().floe_gpu_qgemv_channels_batched(e.handle, x.data_ptr(), x.shape[0], v.data_ptr(),
                                                 _stream(stream)))
    return v


def expert_forward_batched(e: GpuExpert, x, *, v=None, stream=None):
    """expert_forward_sparse for a batch of tokens: x [B, d_hidden] -> y [B, d_hidden]
    (batched up projection on tcgen05, union gate/down records read once; B <= 64)."""
    torch = _torch()
    if x.dim() != 2 or x.shape[1] != e.d_hidden or x.dtype != torch.float32 or not x.is_cuda:
        raise FloeError("expert_forward_batched: x must be a cuda float32 [B, d_hidden]")
    x = x.contiguous()
    y = torch.empty_like(x)
    _check(lib().floe_gpu_expert_forward_batched(e.handle, x.data_ptr(), x.shape[0], y.data_ptr(),
                                                 _ptr(v), _stream(stream)))
    return y


def expert_forward_prefill(e: GpuExpert, x, *, out=None, stream=None):
    """expert_forward_sparse for many tokens (prefill): x [n, d_hidden] -> y [n, d_hidden]
    through dense f16 tensor-core GEMMs with hi/lo splits (any n; the codes and records
    are read once per call)."""
    torch = _torch()
    if x.dim() != 2 or x.shape[1] != e.d_hidden or x.dtype != torch.float32 or not x.is_cuda:
        raise FloeError("expert_forward_prefill: x must be a cuda float32 [n, d_hidden]")
    x = x.contiguous()
    y = torch.empty_like(x) if out is None else out
    _check(lib().floe_gpu_expert_forward_prefill(e.handle, x.data_ptr(), x.shape[0], y.data_ptr(),
                                                 _stream(stream)))
    return y


def dequantize(e: GpuExpert, stream=None):
    """floe::dequantize(up_q) on the device (bit-exact f32)."""
    torch = _torch()
    out = torch.empty(e.d_hidden * e.d_intermediate, dtype=torch.float32, device="cuda")
    _check(lib().floe_gpu_dequantize_up(e.handle, out.data_ptr(), _stream(stream)))
    return out


def predict_mask(e_next: GpuExpert, x_prev, t: float, ws: Workspace, *, kept=None,
                 n_kept=None, stream=None):
    """floe::predict_mask(up_next, d_hidden, x_prev, t) (predictor.cpp:179-189) -> u8 mask."""
    torch = _torch()
    x_prev = _dev_f32(x_prev, e_next.d_hidden, "predict_mask")
    mask = torch.empty(e_next.d_intermediate, dtype=torch.uint8, device=x_prev.device)
    _check(lib().floe_gpu_predict_mask(e_next.handle, ws.handle, x_prev.data_ptr(), float(t),
                                       mask.data_ptr(), _ptr(kept), _ptr(n_kept),
                                       _stream(stream)))
    return mask


class GpuLayer:
    """One compressed MoE block (floe::CompressedLayer + top_k) on the device."""

    def __init__(self, router, mixing, experts: list[GpuExpert], top_k: int,
                 mixing_f16: bool = True):
        """router [E][dh], mixing [dh][dh]: f32 numpy arrays or cuda tensors."""
        if hasattr(router, "data_ptr"):
            router = router.float().contiguous()
        else:
            router = np.ascontiguousarray(router, np.float32)
        if hasattr(mixing, "data_ptr"):
            mixing = mixing.float().contiguous()
        else:
            mixing = np.ascontiguousarray(mixing, np.float32)
        E = len(experts)
        arr = (ct.c_void_p * E)(*[e.handle for e in experts])
        v = LayerHostView(mixing.shape[0], E, top_k, _ptr(router), _ptr(mixing),
                          1 if mixing_f16 else 0, ct.addressof(arr))
        h = ct.c_void_p()
        _check(lib().floe_gpu_layer_create(ct.byref(v), ct.byref(h)))
        self.handle = h.value
        self.experts = experts  # borrowed by the device layer: keep alive
        self.d_hidden = mixing.shape[0]
        self.d_intermediate = experts[0].d_intermediate
        self.n_experts, self.top_k = E, top_k

    @classmethod
    def _adopt(cls, handle, experts, d_hidden, top_k):
        l = cls.__new__(cls)
        l.handle = handle
        l.experts = experts
        l.d_hidden = d_hidden
        l.d_intermediate = experts[0].d_intermediate
        l.n_experts, l.top_k = len(experts), top_k
        return l

    def close(self):
        if getattr(self, "handle", None):
            lib().floe_gpu_layer_destroy(self.handle)
            self.handle = None

    __del__ = close


def layer_forward(layer: GpuLayer, h, ws: Workspace, *, traced: bool = False, out=None,
                  stream=None):
    """floe::layer_forward / layer_forward_traced (model.cpp:145-208)."""
    torch = _torch()
    h = _dev_f32(h, layer.d_hidden, "layer_forward")
    y = torch.empty(layer.d_hidden, dtype=torch.float32, device=h.device) if out is None else out
    tr = None
    if traced:
        k, di = layer.top_k, layer.d_intermediate
        res = dict(block_input=torch.empty(layer.d_hidden, dtype=torch.float32, device=h.device),
                   experts=torch.empty(k, dtype=torch.int32, device=h.device),
                   weights=torch.empty(k, dtype=torch.float32, device=h.device),
                   masks=torch.empty((k, di), dtype=torch.uint8, device=h.device))
        tr = LayerTrace(res["block_input"].data_ptr(), res["experts"].data_ptr(),
                        res["weights"].data_ptr(), res["masks"].data_ptr())
    _check(lib().floe_gpu_layer_forward(layer.handle, ws.handle, h.data_ptr(), y.data_ptr(),
                                        ct.byref(tr) if tr is not None else None,
                                        _stream(stream)))
    if traced:
        res["out"] = y
        return res
    return y


class RecordCacheInfo(ct.Structure):
    _fields_ = [("layers", _U32), ("experts", _U32), ("top_k", _U32), ("d_hidden", _U32),
                ("d_intermediate", _U32), ("bits", _U32), ("group_size", _U32),
                ("mixing_f16", _U32), ("file_bytes", ct.c_uint64)]


def save_record_cache(path: str, layers) -> None:
    """Write the layers as a FLOR record-cache file (include/floe_gpu.h): the
    device-friendly counterpart of FLOQ, f16 gate|down records."""
    arr = (ct.c_void_p * len(layers))(*[l.handle for l in layers])
    _check(lib().floe_gpu_record_cache_save(arr, len(layers), str(path).encode()))


def record_cache_info(path: str) -> dict:
    i = RecordCacheInfo()
    _check(lib().floe_gpu_record_cache_info(str(path).encode(), ct.byref(i)))
    return {f: getattr(i, f) for f, _ in RecordCacheInfo._fields_}


def load_record_cache(path: str, host_records: bool = False) -> list:
    """A FLOR file -> GpuLayers (each owning its experts)."""
    i = record_cache_info(path)
    L, E = i["layers"], i["experts"]
    lh = (ct.c_void_p * L)()
    eh = (ct.c_void_p * (L * E))()
    _check(lib().floe_gpu_record_cache_load(str(path).encode(),
                                            FLOE_VIEW_HOST_RECORDS if host_records else 0, lh, eh))
    layers = []
    for l in range(L):
        ex = [GpuExpert._adopt(eh[l * E + e], i["d_hidden"], i["d_intermediate"], i["bits"],
                               i["group_size"]) for e in range(E)]
        layers.append(GpuLayer._adopt(lh[l], ex, i["d_hidden"], i["top_k"]))
    return layers


class GpuPredictor:
    """floe::InterExpertPredictor on the device: w [layers-1][E][dh], b [layers-1][E]."""

    def __init__(self, w: np.ndarray, b: np.ndarray):
        w = np.ascontiguousarray(w, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        L1, E, dh = w.shape
        h = ct.c_void_p()
        _check(lib().floe_gpu_predictor_create(L1 + 1, E, dh, w.ctypes.data, b.ctypes.data,
                                               ct.byref(h)))
        self.handle = h.value
        self.layers, self.experts, self.d_hidden = L1 + 1, E, dh

    def close(self):
        if getattr(self, "handle", None):
            lib().floe_gpu_predictor_destroy(self.handle)
            self.handle = None

    __del__ = close


def predict_experts(p: GpuPredictor, x, layer: int, count: int, stream=None):
    """floe::predict_experts(p, x, layer, prefetch_count) (predictor.cpp:164-177)."""
    torch = _torch()
    x = _dev_f32(x, p.d_hidden, "predict_experts")
    out = torch.empty(max(count, 1), dtype=torch.int32, device=x.device)
    _check(lib().floe_gpu_predict_experts(p.handle, x.data_ptr(), layer, count, out.data_ptr(),
                                          _stream(stream)))
    return out[:count]


def pack_compact(e: GpuExpert, mask, element_bytes: int = 2, stream=None):
    """pack_compact (offload.cpp:27-53) of the masked channels: (channels [n] u32,
    payload [n * 4 * d_hidden] u8) as cuda tensors."""
    torch = _torch()
    mask = mask.to(torch.uint8).contiguous()
    di, dh = e.d_intermediate, e.d_hidden
    ch = torch.empty(di, dtype=torch.int32, device=mask.device)
    payload = torch.empty(di * 2 * dh * element_bytes, dtype=torch.uint8, device=mask.device)
    n = torch.zeros(1, dtype=torch.int32, device=mask.device)
    _check(lib().floe_gpu_pack_compact(e.handle, mask.data_ptr(), element_bytes, ch.data_ptr(),
                                       payload.data_ptr(), n.data_ptr(), _stream(stream)))
    k = int(n.item())
    return ch[:k], payload[:k * 2 * dh * element_bytes]


def layer_forward_batched(layer: GpuLayer, h, ws: Workspace = None, out=None, stream=None):
    """block_forward (model.cpp:145-169) for a batch: h [n, dh] -> y [n, dh]; with a
    workspace, experts routed few tokens use the fused single-expert kernel."""
    torch = _torch()
    if h.dim() != 2 or h.shape[1] != layer.d_hidden or h.dtype != torch.float32 or not h.is_cuda:
        raise FloeError("layer_forward: dimension mismatch")
    h = h.contiguous()
    y = torch.empty_like(h) if out is None else out
    _check(lib().floe_gpu_layer_forward_batched(layer.handle, ws.handle if ws else None,
                                                h.data_ptr(), h.shape[0], y.data_ptr(),
                                                _stream(stream)))
    return y


def layer_forward_host(layer: GpuLayer, h: np.ndarray, ws: Workspace, out=None, stream=None):
    """Host-buffer layer_forward (H2D, the four kernels, D2H, synchronise)."""
    h = np.ascontiguousarray(h, np.float32)
    if h.size != layer.d_hidden:
        raise FloeError("layer_forward: dimension mismatch")
    y = np.empty(layer.d_hidden, np.float32) if out is None else out
    _check(lib().floe_gpu_layer_forward_host(layer.handle, ws.handle, h.ctypes.data,
                                             y.ctypes.data,
                                             _stream(stream) if stream is not None else 0))
    return y


def gen_normals(seed: int, stream_id: int, n: int, sigma: float = 1.0, sharded: bool = False,
                out=None, stream=None):
    """The reference's Rng(seed, stream) normals (x sigma) generated on the device."""
    torch = _torch()
    out = torch.empty(n, dtype=torch.float32, device="cuda") if out is None else out
    _check(lib().floe_gpu_gen_normals(seed, stream_id, n, float(sigma), 1 if sharded else 0,
                                      out.data_ptr(), _stream(stream)))
    return out


def quantize(x, bits: int, group_size: int, stream=None):
    """floe::quantize on the device -> (codes u8, scales u16-as-int16, zeros) tensors."""
    torch = _torch()
    n = x.numel()
    if group_size == 0 or n % group_size:
        raise FloeError("quantize: group_size must divide element count")
    codes = torch.empty((n * bits + 7) // 8, dtype=torch.uint8, device="cuda")
    scales = torch.empty(n // group_size, dtype=torch.int16, device="cuda")
    zeros = torch.empty(n // group_size, dtype=torch.int16, device="cuda")
    _check(lib().floe_gpu_quantize(x.data_ptr(), n, bits, group_size, codes.data_ptr(),
                                   scales.data_ptr(), zeros.data_ptr(), _stream(stream)))
    return codes, scales, zeros


class OffloadStats(ct.Structure):
    _fields_ = [("tokens", ct.c_uint64), ("records_from_hbm", ct.c_uint64),
                ("records_over_pcie", ct.c_uint64), ("record_bytes", ct.c_uint64),
                ("up_bytes_per_expert", ct.c_uint64), ("promotions", ct.c_uint64),
                ("evictions", ct.c_uint64), ("bytes_promoted", ct.c_uint64),
                ("device_record_bytes", ct.c_uint64),
                ("bytes_demanded", ct.c_uint64), ("bytes_from_cache", ct.c_uint64),
                ("bytes_prefetch_used", ct.c_uint64), ("bytes_sync", ct.c_uint64),
                ("bytes_prefetch_wasted", ct.c_uint64), ("bytes_prefetch_pending", ct.c_uint64),
                ("requests_up", ct.c_uint64), ("requests_channel", ct.c_uint64),
                ("mask_precision", ct.c_double), ("mask_recall", ct.c_double),
                ("mask_samples", ct.c_uint64),
                ("set_precision", ct.c_double), ("set_recall", ct.c_double),
                ("set_samples", ct.c_uint64)]


class Offload:
    """Host-resident decode engine (floe_gpu_offload; SURVEY config 3): the
    layers' experts keep their gate|down records in pinned host memory, an LRU
    of whole experts lives in HBM under `vram_budget` bytes."""

    def __init__(self, layers, vram_budget: int):
        arr = (ct.c_void_p * len(layers))(*[l.handle for l in layers])
        h = ct.c_void_p()
        _check(lib().floe_gpu_offload_create(arr, len(layers), int(vram_budget), ct.byref(h)))
        self.handle = h.value
        self.layers = layers
        self.d_hidden = layers[0].d_hidden
        self.multi_layer = bool(lib().floe_gpu_model_multi_layer(self.handle))

    def close(self):
        if getattr(self, "handle", None):
            lib().floe_gpu_offload_destroy(self.handle)
            self.handle = None

    __del__ = close

    def decode(self, h, ws: Workspace, out=None, stream=None):
        """One token through every layer (h -> y), stream-ordered."""
        torch = _torch()
        h = _dev_f32(h, self.d_hidden, "offload_decode")
        y = torch.empty(self.d_hidden, dtype=torch.float32, device=h.device) if out is None else out
        _check(lib().floe_gpu_offload_decode(self.handle, ws.handle, h.data_ptr(), y.data_ptr(),
                                             _stream(stream)))
        return y

    def decode_replay(self, h, ws: Workspace, out=None, stream=None):
        """One token, each layer on its own recorded block input: h [L, dh] -> y [L, dh]."""
        torch = _torch()
        L = len(self.layers)
        if tuple(h.shape) != (L, self.d_hidden) or h.dtype != torch.float32 or not h.is_cuda:
            raise FloeError("offload_decode_replay: h must be a cuda float32 [layers, d_hidden]")
        h = h.contiguous()
        y = torch.empty_like(h) if out is None else out
        _check(lib().floe_gpu_offload_decode_replay(self.handle, ws.handle, h.data_ptr(),
                                                    y.data_ptr(), _stream(stream)))
        return y

    def set_eval(self, enable: bool = True, predictor=None, count: int = 0):
        """Score the predictors on the decode path: reuse masks (predict_mask of
        layer l's experts from layer l-1's block input) and, with an
        InterExpertPredictor, predict_experts sets (predictor.cpp:206-254)."""
        _check(lib().floe_gpu_offload_set_eval(self.handle, 1 if enable else 0,
                                               predictor.handle if predictor else None,
                                               int(count)))

    def stats(self, stream=None) -> dict:
        st = OffloadStats()
        _check(lib().floe_gpu_offload_stats(self.handle, ct.byref(st), _stream(stream)))
        return {f: getattr(st, f) for f, _ in OffloadStats._fields_}


class GpuModel:
    """A stack of HBM-resident compressed layers (floe::CompressedModel) decoded
    token by token, the reference's run loop (cli.cpp:86-107)."""

    def __init__(self, layers):
        arr = (ct.c_void_p * len(layers))(*[l.handle for l in layers])
        h = ct.c_void_p()
        _check(lib().floe_gpu_model_create(arr, len(layers), ct.byref(h)))
        self.handle = h.value
        self.layers = layers
        self.d_hidden = layers[0].d_hidden
        self.multi_layer = bool(lib().floe_gpu_model_multi_layer(self.handle))

    def close(self):
        if getattr(self, "handle", None):
            lib().floe_gpu_model_destroy(self.handle)
            self.handle = None

    __del__ = close

    def decode(self, h, ws: Workspace, out=None, replay: bool = False, stream=None):
        """replay=False: h [dh] -> y [dh] through every layer.  replay=True: h [L, dh]
        -> y [L, dh], layer l on its own block input."""
        torch = _torch()
        shape = (len(self.layers), self.d_hidden) if replay else (self.d_hidden,)
        if tuple(h.shape) != shape or h.dtype != torch.float32 or not h.is_cuda:
            raise FloeError(f"model_decode: h must be a cuda float32 {shape}")
        h = h.contiguous()
        y = torch.empty_like(h) if out is None else out
        _check(lib().floe_gpu_model_decode(self.handle, ws.handle, h.data_ptr(), y.data_ptr(),
                                           1 if replay else 0, _stream(stream)))
        return y

    def decode_host(self, h: np.ndarray, ws: Workspace, out=None, replay: bool = False,
                    stream=None):
        h = np.ascontiguousarray(h, np.float32)
        y = np.empty_like(h) if out is None else out
        _check(lib().floe_gpu_model_decode_host(self.handle, ws.handle, h.ctypes.data,
                                                y.ctypes.data, 1 if replay else 0,
                                                _stream(stream) if stream is not None else 0))
        return y


class GpuCalib:
    """collect_stats + calibrate_model on the device (model.cpp:242-330): one
    reservoir per (layer, expert), fed layer by layer with dense float layers."""

    def __init__(self, layers: int, experts: int, d_hidden: int, d_intermediate: int, seed: int,
                 sample_cap: int = 1 << 16):
        h = ct.c_void_p()
        _check(lib().floe_gpu_calib_create(layers, experts, d_hidden, d_intermediate, seed,
                                           sample_cap, ct.byref(h)))
        self.handle = h.value
        self.layers, self.experts, self.d_hidden = layers, experts, d_hidden

    def close(self):
        if getattr(self, "handle", None):
            lib().floe_gpu_calib_destroy(self.handle)
            self.handle = None

    __del__ = close

    def layer(self, layer: int, router, mixing, gate, up, down_t, top_k: int, h,
              drift_scale: float = 1.0, want_next: bool = True, stream=None):
        """One layer of collect_stats over tokens h [T, dh] (device f32); gate/up/down_t
        are lists of E device f32 tensors [di, dh].  Returns the next layer's inputs."""
        torch = _torch()
        h = h.contiguous()
        T = h.shape[0]
        arr = ct.c_void_p * len(gate)
        g = arr(*[t.data_ptr() for t in gate])
        u = arr(*[t.data_ptr() for t in up])
        d = arr(*[t.data_ptr() for t in down_t])
        v = FloatLayerView(router.data_ptr(), mixing.data_ptr(), ct.addressof(g), ct.addressof(u),
                           ct.addressof(d))
        nxt = torch.empty_like(h) if want_next else None
        _check(lib().floe_gpu_calib_layer(self.handle, layer, ct.byref(v), top_k,
                                          float(drift_scale), h.data_ptr(),
                                          nxt.data_ptr() if nxt is not None else None, T,
                                          _stream(stream)))
        return nxt

    def thresholds(self, k: float) -> np.ndarray:
        out = np.empty(self.layers * self.experts, np.float32)
        _check(lib().floe_gpu_calib_thresholds(self.handle, float(k), out.ctypes.data))
        return out.reshape(self.layers, self.experts)
