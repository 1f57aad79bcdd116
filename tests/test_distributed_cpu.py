"""Multi-process (gloo, world_size 2 and 4) CPU tests of the time-sharded decomposition:
the NCCL-id broadcast used by the bootstrap, and a numpy model of the four-step time FFT whose
index maps (cyclic steps, chunk positions, slot -> frequency) are the ones the kernels use.
The model exchanges its chunks with a real torch.distributed all_to_all between processes."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bitrev(x, bits):
    return int(format(x, f"0{bits}b")[::-1], 2) if bits else 0


def _worker(rank, world, port, L, alpha, q):
    import torch
    import torch.distributed as dist

    from paper_2103_12571_b200.distributed import broadcast_bytes, chunk_positions, local_steps, slot_frequency
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # 1. id broadcast: everyone gets rank 0's bytes
        payload = bytes(range(128)) if rank == 0 else None
        got = broadcast_bytes(payload)
        ok_bcast = got == bytes(range(128))

        # 2. four-step forward time DFT of alpha^{l/L} r_l over a cyclic distribution
        rng = np.random.default_rng(7)
        C = 3
        r = rng.standard_normal((L, C)) + 1j * rng.standard_normal((L, C))   # global data (same on all)
        Ll = L // world
        Lc = Ll // world
        steps = local_steps(rank, world, L)
        loc = r[steps] * (alpha ** (steps / L))[:, None]
        y = np.fft.fft(loc, axis=0)                                          # local Ll-point FFT
        bits = Ll.bit_length() - 1
        br = np.array([_bitrev(p, bits) for p in range(Ll)])
        y = y[br]                                                            # bit-reversed positions
        y = y * np.exp(-2j * np.pi * rank * br / L)[:, None]                  # four-step twiddle
        send = np.concatenate([y[chunk_positions(d, world, L)] for d in range(world)])
        sendt = torch.from_numpy(np.ascontiguousarray(send).view(np.float64).copy())
        recvt = torch.empty_like(sendt)
        dist.all_to_all_single(recvt, sendt)
        recv = recvt.numpy().view(np.complex128).reshape(world, Lc, C)      # [src g][pl][c]
        # cross-rank P-point DFT: x_{kappa + Ll q} = sum_g e^{-2 pi i g q / P} y_g
        W = np.exp(-2j * np.pi * np.outer(np.arange(world), np.arange(world)) / world)
        x = np.einsum("qg,gpc->qpc", W, recv).reshape(world * Lc, C)         # slot = q*Lc + pl
        ref = np.fft.fft(r * (alpha ** (np.arange(L) / L))[:, None], axis=0)
        ks = [slot_frequency(rank, world, L, s) for s in range(Ll)]
        err = float(np.abs(x - ref[ks]).max() / np.abs(ref).max())
        q.put((rank, ok_bcast, err, sorted(ks)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,L", [(2, 8), (2, 64), (4, 64)])
def test_four_step_over_gloo(world, L):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, L, 0.37, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    allk = []
    for rank, ok, err, ks in res:
        assert ok, rank
        assert err < 1e-13, (rank, err)
        allk += ks
    assert sorted(allk) == list(range(L))   # every frequency owned exactly once


def test_index_maps_match_library_convention():
    """slot_frequency is the map pint_set_alpha_schedule uses for P > 1 (pint_abi.cpp)."""
    from paper_2103_12571_b200.distributed import slot_frequency
    for world, L in [(2, 8), (4, 32), (8, 512)]:
        seen = set()
        for rank in range(world):
            for s in range(L // world):
                seen.add(slot_frequency(rank, world, L, s))
        assert seen == set(range(L))


def _band_worker(rank, world, port, L, q):
    """The overlapped schedule's exchange: band b of every peer chunk (chunk slots pl in band) as a
    separate all-to-all; the cross-rank DFT of each band only needs that band; assembling the bands
    gives the unbanded result, and the bands' slot lists partition the local slots."""
    import torch
    import torch.distributed as dist

    from paper_2103_12571_b200.distributed import band_slots, bands, chunk_positions
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(11 + rank)
        Ll, C = L // world, 5
        Lc = Ll // world
        y = rng.standard_normal((Ll, C)) + 1j * rng.standard_normal((Ll, C))   # this rank's positions
        send = np.concatenate([y[chunk_positions(d, world, L)] for d in range(world)])   # [d][pl][c]
        full = torch.empty(send.size * 2, dtype=torch.float64)
        dist.all_to_all_single(full, torch.from_numpy(np.ascontiguousarray(send).view(np.float64).copy()))
        full = full.numpy().view(np.complex128).reshape(world, Lc, C)
        B = bands(world, L)
        nb = Lc // B
        got = np.zeros_like(full)
        for b in range(B):
            # contiguous band slice of every chunk (the offsets nccl_alltoall uses)
            part = np.ascontiguousarray(send.reshape(world, Lc, C)[:, b * nb:(b + 1) * nb])
            rt = torch.empty(part.size * 2, dtype=torch.float64)
            dist.all_to_all_single(rt, torch.from_numpy(part.view(np.float64).copy()))
            got[:, b * nb:(b + 1) * nb] = rt.numpy().view(np.complex128).reshape(world, nb, C)
        slots = np.concatenate([band_slots(world, L, B, b) for b in range(B)])
        q.put((rank, float(np.abs(got - full).max()), sorted(slots.tolist()) == list(range(Ll)), B))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,L", [(2, 32), (4, 64), (2, 8)])
def test_banded_alltoall_over_gloo(world, L):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_band_worker, args=(r, world, port, L, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, err, partition, B in res:
        assert err == 0.0 and partition, (rank, err, partition, B)
