"""Multi-GPU NLEM: one process per GPU, the image split into contiguous row bands.

Every output pixel is independent, so a rank needs only its band plus a
halo of S/2 + k/2 rows (13 for S=21, k=7) on each side; window clipping and patch
mirroring use GLOBAL image coordinates inside the kernel (nlem_denoise_rows), so the
concatenated bands are bitwise identical to the single-GPU result.  No collective runs
on the data path; torch.distributed (NCCL on GPUs, gloo on CPU) is used only for the
optional final gather and for timing barriers.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Tuple

import numpy as np


def band_partition(rows: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous bands [(row0, nrows)] of ceil(rows/world) rows (the last may be short)."""
    per = (rows + world - 1) // world
    out = []
    for r in range(world):
        r0 = min(rows, r * per)
        out.append((r0, min(rows, r0 + per) - r0))
    return out


def input_rows(rows: int, r0: int, nrows: int, halo: int) -> Tuple[int, int]:
    """Input rows [i0, i1) a band reads: its rows plus `halo` on each side, clipped."""
    return max(0, r0 - halo), min(rows, r0 + nrows + halo)


def halo_for(search: int, patch: int) -> int:
    return search // 2 + patch // 2


BandFn = Callable[[np.ndarray, int, int, int, int, int], np.ndarray]


def gpu_band_fn(params, device: int = 0) -> BandFn:
    """The GPU compute for one band through the host-buffer C-ABI entry."""
    from . import api

    def fn(in_rows_arr, in_row0, rows, cols, out_row0, out_rows):
        return api.nlem_denoise_rows_host(in_rows_arr, in_row0, rows, cols, out_row0, out_rows,
                                          params, device=device)

    return fn


def denoise_bands(noisy: np.ndarray, search: int, patch: int, rank: int, world: int,
                  band_fn: BandFn, group=None, gather: bool = True) -> Optional[np.ndarray]:
    """Run this rank's band; with gather=True rank 0 returns the full image (others None),
    else every rank returns its own band."""
    rows, cols = noisy.shape
    r0, nrows = band_partition(rows, world)[rank]
    i0, i1 = input_rows(rows, r0, nrows, halo_for(search, patch))
    band = band_fn(np.ascontiguousarray(noisy[i0:i1], dtype=np.float32), i0, rows, cols, r0, nrows)
    if not gather or world == 1:
        return band
    import torch
    import torch.distributed as dist

    parts = [None] * world
    dist.all_gather_object(parts, np.asarray(band), group=group)
    if rank != 0:
        return None
    return np.concatenate(parts, axis=0)
