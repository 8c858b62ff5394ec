"""Multi-GPU sweeps: ray sharding across ranks + one all-reduce of the accumulators.

One process per GPU (torch.distributed, NCCL over NVLink / NVSwitch).  Every
rank holds a replica of the scene (uploaded + BVH built on its own GPU) and
traces a disjoint range of EVERY incidence's launch entries,

    stripes k = rank, rank + world, rank + 2 world, ... of S dispatch
    indices each, S ~ entries / (32 world) rounded up to 1024    (shard_stripes)

of the dispatch order (4-row bands of strata, trace.cu locate(); the same
integer partition the C ABI applies in mcsbr_gpu_trace_device, capi.cu
plan_job).  Interleaving balances the ranks whatever the target's silhouette
(contiguous shards put an airframe's whole silhouette on the middle ranks),
and the counter-RNG keys (seed, cell, sample) -- hence every path -- are independent of the GPU count.  The raw complex
phasor sums ([n_inc][n_rx][nf][4] fp64) and the uint64 counters are then
summed with one all-reduce each; the j k0 / (2 sqrt(pi)) finalisation runs
on the host.  This mirrors the reference's own fixed-order block merge
(proj/src/solver_mc.cpp:212-224) with ranks in place of blocks; the result
agrees with the single-GPU sweep to fp64 rounding (sum order only).

The payload is small (c5: 128 x 128 x 4 complex = 1 MiB), so the collective
is latency-bound and a plain NCCL all-reduce is the right tool here; there is
no per-tile exchange to fuse with compute.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi as A


def shard_stripes(entries: int, rank: int, world: int) -> list[tuple[int, int]]:
    """Dispatch-index ranges of `rank` (identical to capi.cu plan_job): one
    range [0, entries) for world 1, else stripes of S indices, stripe k to
    rank k mod world, S = max(1024, ceil(entries / (32 world)) rounded up to
    a multiple of 1024)."""
    if world == 1:
        return [(0, entries)] if entries else []
    s = -(-entries // (32 * world))
    s = max(1024, -(-s // 1024) * 1024)
    n = -(-entries // s)
    return [(k * s, min(entries, (k + 1) * s)) for k in range(rank, n, world)]


def allreduce_finalize(sums, counters, freqs, n: int, group=None):
    """Sum raw accumulators / counters over the process group, finalize on host.

    sums: torch float64 tensor with n * nf * 8 elements ([n][nf][4] complex,
    the device layout), or for MCSBR_REDUCE_EXACT jobs an int64 tensor of
    n * nf * 8 * MCSBR_EXACT_LIMBS limbs (summed exactly by the integer
    all-reduce); counters: torch int64 tensor of MCSBR_COUNTER_WORDS.
    Works with any backend (NCCL for CUDA tensors, gloo for CPU tensors).
    Returns (values complex [n][4][nf], mcsbr_stats).
    """
    import torch
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        # word 6 holds fault BITS (atomicOr on the device) and word 7 the
        # deepest bounce round (atomicMax): they are combined with a bitwise
        # OR and a max over ranks; everything else is a sum
        special = counters[6:8].clone()
        counters[6:8] = 0
        dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(counters, op=dist.ReduceOp.SUM, group=group)
        world = dist.get_world_size(group)
        gathered = [torch.zeros_like(special) for _ in range(world)]
        dist.all_gather(gathered, special, group=group)
        fault, rounds = 0, 0
        for g in gathered:
            fault |= int(g[0].item())
            rounds = max(rounds, int(g[1].item()))
        counters[6] = fault
        counters[7] = rounds
    freqs = np.ascontiguousarray(np.asarray(freqs, dtype=np.float64).reshape(-1))
    nf = len(freqs)
    values = np.zeros((n, 4, nf, 2), dtype=np.float64)
    L = A.lib()
    if sums.dtype == torch.int64:  # MCSBR_REDUCE_EXACT: integer limbs, summed exactly over ranks
        raw = np.ascontiguousarray(sums.detach().cpu().numpy())
        A.check(L.mcsbr_gpu_finalize_exact(raw.ctypes.data_as(C.POINTER(C.c_int64)), n,
                                           freqs.ctypes.data_as(C.POINTER(C.c_double)), nf,
                                           values.ctypes.data_as(C.POINTER(C.c_double))))
    else:
        raw = np.ascontiguousarray(sums.detach().to("cpu", torch.float64).numpy())
        A.check(L.mcsbr_gpu_finalize(raw.ctypes.data_as(C.POINTER(C.c_double)), n,
                                     freqs.ctypes.data_as(C.POINTER(C.c_double)), nf,
                                     values.ctypes.data_as(C.POINTER(C.c_double))))
    cnt = np.ascontiguousarray(counters.detach().cpu().numpy().astype(np.uint64))
    st = A.Stats()
    rc = L.mcsbr_gpu_decode_counters(cnt.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(st))
    if rc != 0:
        A.check(rc)
    return values[..., 0] + 1j * values[..., 1], st


def sweep_sharded(scene, incidences, receivers, frequencies, config, occlusion_enabled=True,
                  group=None, stream=None):
    """Distributed counterpart of solver.estimate_batch.

    Each rank traces its shard on its own GPU (scene.device) into device
    buffers, then the buffers are all-reduced (NCCL) and finalized.  Every
    rank returns the full result.  `incidences` / `receivers` as in
    estimate_batch.
    """
    import torch
    import torch.distributed as dist

    rank, world = 0, 1
    if dist.is_available() and dist.is_initialized():
        rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = torch.device("cuda", scene.device)
    freqs = np.ascontiguousarray(np.asarray(frequencies, dtype=np.float64).reshape(-1))
    n_inc = len(incidences)
    n_rx = len(receivers[0])
    inc_arr = (A.Incidence * n_inc)(*[e.incidence(spw) for e, spw in incidences])
    rx_arr = (A.Receiver * (n_inc * n_rx))(*[r.receiver() for rl in receivers for r in rl])
    exact = int(config.reduction) == A.MCSBR_REDUCE_EXACT
    sums = (torch.zeros(n_inc * n_rx * len(freqs) * 8 * A.MCSBR_EXACT_LIMBS, dtype=torch.int64, device=dev) if exact
            else torch.zeros(n_inc * n_rx * len(freqs) * 8, dtype=torch.float64, device=dev))
    counters = torch.zeros(A.MCSBR_COUNTER_WORDS, dtype=torch.int64, device=dev)
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    cfg = config.to_c()
    A.check(A.lib().mcsbr_gpu_trace_device(
        scene.handle, inc_arr, n_inc, rx_arr, n_rx, 1 if occlusion_enabled else 0,
        freqs.ctypes.data_as(C.POINTER(C.c_double)), len(freqs), C.byref(cfg), rank, world,
        C.c_void_p(sums.data_ptr()), C.c_void_p(counters.data_ptr()), C.c_void_p(st.cuda_stream)))
    values, stats = allreduce_finalize(sums, counters, freqs, n_inc * n_rx, group)
    return values.reshape(n_inc, n_rx, 4, len(freqs)), stats
