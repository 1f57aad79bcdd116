"""Multi-process plumbing for the time-sharded path (one process per GPU, torchrun).

torch.distributed is used only to bootstrap: rank 0 asks libpint for a 128-byte NCCL unique id
and it is broadcast over the default process group (gloo on CPU tests, nccl on GPUs); every
rank then creates its own libpint context, which owns the NCCL communicator used inside the
iteration (all-to-all + ring halo on the library's stream).

The index maps below mirror the ones the kernels use and are exercised by the CPU
multi-process tests (tests/test_distributed_cpu.py).
"""
from __future__ import annotations

import os
from typing import Tuple

import numpy as np


def env_rank() -> Tuple[int, int, int]:
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def local_steps(rank: int, nranks: int, L: int) -> np.ndarray:
    """Global steps owned by `rank` under the cyclic distribution l = rank + nranks * j."""
    return np.arange(rank, L, nranks)


def chunk_positions(dest: int, nranks: int, L: int) -> np.ndarray:
    """Local FFT positions p (bit-reversed kappa) sent to rank `dest` in the all-to-all."""
    Lc = L // nranks // nranks
    return np.arange(dest * Lc, (dest + 1) * Lc)


def slot_frequency(rank: int, nranks: int, L: int, slot: int) -> int:
    """Global time frequency k held at local frequency slot `slot` after the cross-rank DFT:
    slot = q * Lc + pl  ->  k = bitrev_{L/P}(rank * Lc + pl) + (L/P) q."""
    Ll = L // nranks
    Lc = Ll // nranks
    q, pl = divmod(slot, Lc)
    bits = Ll.bit_length() - 1
    kappa = int(format(rank * Lc + pl, f"0{bits}b")[::-1], 2) if bits > 0 else 0
    return kappa + Ll * q


def bands(nranks: int, L: int, dim: int = 2) -> int:
    """Number of bands of the overlapped schedule (pint_create: 4 in 2-D if L/P^2 allows it)."""
    Lc = L // nranks // nranks
    B = 4 if dim == 2 else 1
    while B > 1 and Lc % B:
        B //= 2
    return B


def band_slots(nranks: int, L: int, B: int, b: int) -> np.ndarray:
    """Local frequency slots solved in band b: {q Lc + pl : q < P, pl in [b nb, (b+1) nb)}, the
    order of the device list at work + off_band (pint_abi.cpp)."""
    Lc = L // nranks // nranks
    nb = Lc // B
    return np.array([q * Lc + pl for q in range(nranks) for pl in range(b * nb, (b + 1) * nb)])


def broadcast_bytes(payload: bytes | None, src: int = 0, nbytes: int = 128) -> bytes:
    """Broadcast `nbytes` bytes from rank `src` over the default torch.distributed group."""
    import torch
    import torch.distributed as dist
    backend = dist.get_backend()
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
    if dist.get_rank() == src:
        assert payload is not None and len(payload) == nbytes
        t.copy_(torch.frombuffer(bytearray(payload), dtype=torch.uint8))
    dist.broadcast(t, src)
    return bytes(t.cpu().numpy().tobytes())


def sharded_solver(problem, u0: np.ndarray, device: int | None = None):
    """Creates this rank's libpint context of an NCCL-sharded problem (call inside torchrun after
    torch.distributed.init_process_group)."""
    import torch.distributed as dist

    import paper_2103_12571_b200 as P
    rank, world = dist.get_rank(), dist.get_world_size()
    if world == 1:
        return P.Solver(problem, u0, device=device or 0)
    uid = P.nccl_unique_id() if rank == 0 else None
    uid = broadcast_bytes(uid)
    return P.Solver(problem, u0, device=device if device is not None else env_rank()[2], rank=rank, nranks=world,
                    nccl_id=uid)
