"""Expert-parallel MoE layer: the experts of
a layer are sharded over the ranks of a process group (rank r owns experts
[r*E/W, (r+1)*E/W)); every rank routes its own tokens, dispatches (token,
expert) pairs to the owning ranks with an all-to-all, runs its experts on what
it received, and gets the outputs back with the reverse all-to-all; the
combine happens on the source rank.

Per token the arithmetic is the reference's block (model.cpp:145-169):
  u = h + mixing h;  logits = router u;  top_k (ties to the lower index,
  selection in ascending expert order, la.cpp:48-61);  w = softmax of the
  selected logits (la.cpp:37-46);  y = u + sum_j w_j expert_j(u) in ascending
  expert order.
The mixing product for a token batch is a plain GEMM: with an f16 mixing
matrix (the device layers' format) it runs on the tensor cores as two f16
GEMMs with f32 accumulation over the hi and lo halves of the (row-scaled)
activations; the router product is a small f32 GEMM.  The experts run through
`expert_fn` -- on the GPU `batched_expert_fn`: the prefill expert forward
(dense f16 tensor-core GEMMs, codes and records read once per expert) for
experts with many tokens, the tcgen05 batched forward or the fused
single-token kernel for few.  The collectives are
NCCL over NVLink on GPUs (gloo in the CPU tests).  Fusing dispatch/combine
with the expert kernels over peer memory is the next step; this module is the
reference-semantics baseline for it.
"""
from __future__ import annotations

from typing import Callable, Optional


def route_topk(torch, logits, k: int):
    """top_k with ties to the lower index, selection in ascending expert
    order, softmax over the selected logits (la.cpp:37-61)."""
    order = torch.sort(-logits, dim=1, stable=True).indices[:, :k]
    sel = torch.sort(order, dim=1).values
    lg = torch.gather(logits, 1, sel)
    mx = lg.max(dim=1, keepdim=True).values
    ex = torch.exp(lg - mx)
    return sel, ex / ex.sum(dim=1, keepdim=True)


def mixing_product(torch, h, mixing):
    """h @ mixing^T.  f16 mixing on a GPU: h scaled per row by a power of two,
    split into f16 hi + lo, two tensor-core GEMMs with f32 output (exact up to
    the f32 accumulation); otherwise a plain f32 GEMM."""
    if mixing.dtype != torch.float16 or not h.is_cuda:
        return h @ mixing.t().to(h.dtype)
    mx = h.abs().amax(dim=1, keepdim=True)
    e = torch.frexp(torch.where(torch.isfinite(mx) & (mx > 0), mx, torch.ones_like(mx)))[1]
    s = torch.ldexp(torch.ones_like(mx), -e)
    hs = h * s
    hi = hs.half()
    lo = (hs - hi.float()).half()
    mt = mixing.t()
    out = torch.mm(hi, mt, out_dtype=torch.float32)
    out += torch.mm(lo, mt, out_dtype=torch.float32)
    return out / s


def _a2a(torch, dist, group, x, out_splits, in_splits):
    out = x.new_empty((sum(out_splits),) + tuple(x.shape[1:]))
    dist.all_to_all_single(out, x.contiguous(), out_splits, in_splits, group=group)
    return out


def ep_moe_layer(h, router, mixing, top_k: int, expert_fn: Callable, n_experts: int,
                 group=None):
    """One expert-parallel MoE layer over this rank's tokens h [T, dh].

    expert_fn(e, X [n, dh]) -> Y [n, dh] runs local expert e (global index).
    Returns y [T, dh] and the routing (sel [T, k], w [T, k])."""
    import torch
    import torch.distributed as dist

    dist_on = dist.is_available() and dist.is_initialized()
    world = dist.get_world_size(group) if dist_on else 1
    if n_experts % world:
        raise ValueError("ep_moe_layer: experts must divide evenly over the ranks")
    per_rank = n_experts // world
    u = h + mixing_product(torch, h, mixing)    # block input (model.cpp:150-152)
    sel, w = route_topk(torch, u @ router.t(), top_k)
    T = h.shape[0]
    pair_tok = torch.arange(T, device=h.device).repeat_interleave(top_k)
    pair_exp = sel.reshape(-1)
    dest = pair_exp // per_rank
    order = torch.sort(dest, stable=True).indices        # pairs grouped by owner
    send = torch.bincount(dest, minlength=world)
    x_send = u[pair_tok[order]]
    e_send = pair_exp[order]
    if world > 1:
        recv = torch.empty_like(send)
        dist.all_to_all_single(recv, send, group=group)  # counts
        s_list, r_list = send.tolist(), recv.tolist()
        x_recv = _a2a(torch, dist, group, x_send, r_list, s_list)
        e_recv = _a2a(torch, dist, group, e_send, r_list, s_list)
    else:
        x_recv, e_recv = x_send, e_send
    # group the received rows by expert (one host sync for the counts), run
    # each local expert on a contiguous slice, scatter back
    perm = torch.sort(e_recv, stable=True).indices
    x_sorted = x_recv[perm]
    counts = torch.bincount(e_recv, minlength=n_experts).tolist()
    out_sorted = torch.empty_like(x_sorted)
    off = 0
    for e, c in enumerate(counts):
        if c:
            out_sorted[off:off + c] = expert_fn(e, x_sorted[off:off + c])
            off += c
    out = torch.empty_like(x_recv)
    out[perm] = out_sorted
    back = _a2a(torch, dist, group, out, s_list, r_list) if world > 1 else out
    contrib = torch.empty_like(back)
    contrib[order] = back
    contrib = contrib.view(T, top_k, h.shape[1])
    y = u.clone()
    for j in range(top_k):                      # ascending expert order (model.cpp:160-166)
        y = y + w[:, j:j + 1] * contrib[:, j]
    return y, sel, w


def batched_expert_fn(experts, first_expert: int = 0, chunk: int = 64, small: int = 7,
                      prefill_min: int = 8):
    """expert_fn over GpuExpert objects on this rank: an expert with at least
    `prefill_min` tokens runs them all through the prefill expert forward
    (exact batched up projection or dequantized f16 hi/lo GEMM, dense f16
    gate/down GEMMs: codes and records read once, ~0.18 ms up to 64 tokens);
    at most `small` tokens go one by one through the single-token fused kernel
    (~25 us each); in between, the batched expert forward in chunks of <= 64.
    experts[i] is global expert first_expert + i."""
    from . import _abi
    wss = {}

    def fn(e: int, X):
        import torch
        ex = experts[e - first_expert]
        n = X.shape[0]
        if n == 0:
            return X.clone()
        if n <= small:
            key = (ex.d_hidden, ex.d_intermediate)
            if key not in wss:
                wss[key] = _abi.Workspace(ex.d_hidden, ex.d_intermediate, 1)
            return torch.stack([_abi.expert_forward_sparse(ex, X[i], wss[key]) for i in range(n)])
        if n >= prefill_min:
            return _abi.expert_forward_prefill(ex, X)
        parts = [_abi.expert_forward_batched(ex, X[i:i + chunk]) for i in range(0, n, chunk)]
        return torch.cat(parts, dim=0)

    return fn
