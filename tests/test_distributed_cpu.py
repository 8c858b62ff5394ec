"""CPU, world_size 2 (gloo): the multi-rank reduction path.

Each rank computes the raw accumulators of ITS launch-entry shard
(distributed.shard_stripes, the partition mcsbr_gpu_trace_device applies) with
the oracle standing in for the device trace, then runs the product's
allreduce_finalize (the same code the NCCL path runs).  The reduced result
must equal the single-process estimate to fp64 rounding, and the counters
must add up exactly.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2511_07586_b200 as M
from paper_2511_07586_b200 import distributed as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case():
    sd = M.make_builtin_scene("glass_cube", {"eps_r": 2.25, "size_m": 1.0})
    exc = M.bistatic_excitation(20.0, 40.0, 60.0, 10.0)
    freqs = np.linspace(1e9, 3e9, 4)
    cfg = M.McConfig(strata_per_wavelength=6, samples_per_stratum=2, seed=99,
                     roulette=M.RouletteConfig(enabled=True))
    return sd, exc, freqs, cfg


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sd, exc, freqs, cfg = _case()
        ps = oracle.port_scene(sd)
        _, _, total = oracle.port_estimate_range(ps, exc.to_c(), freqs, cfg.to_c(), 0, 0)
        stripes = D.shard_stripes(total, rank, world)
        assert stripes, "the test case gives every rank a stripe"
        sums = None
        counters = torch.zeros(256, dtype=torch.int64)
        for b, e in stripes:
            raw, st, _ = oracle.port_estimate_range(ps, exc.to_c(), freqs, cfg.to_c(), b, e)
            part = torch.from_numpy(raw.reshape(-1).copy())
            sums = part if sums is None else sums + part
            counters[0] += st.rays_launched
            counters[2] += st.contributions
            counters[4] += st.cap_kills
            for i in range(64):
                counters[8 + i] += st.rays_per_bounce[i]
                counters[72 + i] += st.roulette_candidates[i]
                counters[136 + i] += st.roulette_survivors[i]
        values, stats = D.allreduce_finalize(sums, counters, freqs, 1)
        if rank == 0:
            np.save(out, values.reshape(4, len(freqs)))
            np.save(out + ".cnt.npy", np.array([stats.rays_launched, stats.contributions,
                                                 stats.cap_kills, stats.segments_traced]))
    finally:
        dist.destroy_process_group()


def test_shard_stripes_partition():
    """The stripes of all ranks tile [0, entries) exactly once, and every
    rank holds a share within one stripe of the mean."""
    for entries in (0, 1, 7, 1000, 4_008_004, 16_777_216, 10**9 + 3):
        for world in (1, 2, 3, 8):
            per = [D.shard_stripes(entries, k, world) for k in range(world)]
            allr = sorted(r for p in per for r in p)
            assert sum(e - b for b, e in allr) == entries
            assert all(allr[k][1] == allr[k + 1][0] for k in range(len(allr) - 1))
            if allr:
                assert allr[0][0] == 0 and allr[-1][1] == entries
                width = max(e - b for b, e in allr)
                share = [sum(e - b for b, e in p) for p in per]
                assert max(share) - min(share) <= width


@pytest.mark.timeout(300)
def test_two_rank_gloo_reduction_matches_single_process(tmp_path):
    out = str(tmp_path / "vals.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    cnt = np.load(out + ".cnt.npy")
    sd, exc, freqs, cfg = _case()
    ref = oracle.port_estimate(oracle.port_scene(sd), exc.to_c(), freqs, cfg.to_c())
    scale = np.max(np.abs(ref["values"]))
    assert np.max(np.abs(got - ref["values"])) <= 1e-12 * scale
    st = ref["stats"]
    assert list(cnt) == [st.rays_launched, st.contributions, st.cap_kills, st.segments_traced]


def _fault_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sums = torch.zeros(8, dtype=torch.float64)
        counters = torch.zeros(256, dtype=torch.int64)
        counters[0] = 10 + rank
        counters[6] = 1 << rank        # rank 0: fresnel domain, rank 1: non-transverse field
        counters[7] = 3 + 2 * rank     # deepest round seen: 3 and 5
        msg = ""
        try:
            D.allreduce_finalize(sums, counters, [1e9], 1)
        except Exception as e:  # noqa: BLE001 - the EDEVICE error is the point
            msg = str(e)
        if rank == 0:
            np.save(out, np.array([int(counters[0]), int(counters[6]), int(counters[7])]))
            with open(out + ".msg", "w") as f:
                f.write(msg)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_fault_bits_are_ored_and_rounds_max_reduced(tmp_path):
    """the fault word carries bit flags (device atomicOr) and word 7
    the deepest bounce round (atomicMax); ranks raising different faults must
    all be reported, and the round count must not be summed."""
    out = str(tmp_path / "cnt.npy")
    mp.spawn(_fault_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    launched, fault, rounds = np.load(out)
    assert launched == 21 and fault == 3 and rounds == 5
    msg = open(out + ".msg").read()
    assert "fresnel" in msg and "transverse" in msg, msg
