"""B200-native FloE compressed-expert FFN path (arXiv 2505.05950).

The product is ``libfloe_b200.so`` (sm_100a kernels + the C ABI declared in
``include/floe_gpu.h``).  This package is a thin ctypes front end over that
ABI, named after the reference's own API (``floe::expert_forward_sparse``,
``floe::layer_forward``, ``floe::predict_mask``, ``floe::predict_experts``,
``floe::qgemv_channels``, ``floe::dequantize``) so the parity tests read like
the reference's tests.  C++ callers use ``include/floe_b200.hpp`` instead.

There is no CPU fallback: importing works anywhere (so the ABI can be
inspected), but every compute call raises ``FloeError`` unless the library is
built and an sm_100 GPU is present.
"""
from ._abi import (  # noqa: F401
    FloeError,
    GpuCalib,
    GpuExpert,
    GpuLayer,
    GpuModel,
    GpuPredictor,
    Offload,
    Workspace,
    abi_version,
    dequantize,
    device_info,
    expert_forward_sparse,
    gen_normals,
    exported_symbols,
    layer_forward,
    layer_forward_batched,
    layer_forward_host,
    pack_compact,
    lib,
    library_path,
    predict_experts,
    predict_mask,
    qgemv_channels,
    qgemv_channels_batched,
    expert_forward_batched,
    expert_forward_prefill,
    quantize,
    save_record_cache,
    load_record_cache,
    record_cache_info,
)

__all__ = ["FloeError", "GpuCalib", "GpuExpert", "GpuLayer", "GpuModel", "GpuPredictor", "Offload", "Workspace",
           "abi_version", "dequantize", "device_info", "expert_forward_sparse",
           "exported_symbols", "layer_forward", "layer_forward_batched", "lib", "library_path", "predict_experts",
           "predict_mask", "qgemv_channels", "qgemv_channels_batched", "expert_forward_batched", "expert_forward_prefill", "gen_normals", "layer_forward_host", "pack_compact",
           "quantize", "save_record_cache", "load_record_cache", "record_cache_info"]
