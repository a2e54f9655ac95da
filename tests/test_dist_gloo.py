"""World-size-2 (gloo, CPU) tests of the multi-GPU row-band path: band partition, halo,
global-coordinate geometry and the final gather, with the FP64 oracle computing each
band (restricted rows) in place of the GPU kernel.  The concatenated result must equal the
single-process oracle image exactly."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1501_03879_b200 import dist as D

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_partition_covers_image():
    for rows in (1, 5, 13, 96, 4096):
        for world in (1, 2, 3, 4, 8):
            bands = D.band_partition(rows, world)
            assert sum(n for _, n in bands) == rows
            nxt = 0
            for r0, n in bands:
                if n:
                    assert r0 == nxt
                    nxt = r0 + n
    assert D.halo_for(21, 7) == 13
    assert D.input_rows(4096, 1024, 1024, 13) == (1011, 2061)
    assert D.input_rows(4096, 0, 1024, 13) == (0, 1037)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, noisy, out_path):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from oracle import oracle as O

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = O.make_params(search=7, patch=3, h=40.0, solver="admm", solver_iters=5, mu=1.0,
                      init_mode="nlm", threads=1)

    def band_fn(in_rows_arr, in_row0, rows, cols, out_row0, out_rows):
        # the oracle sees only this rank's input rows, placed at their global offsets; rows
        # outside the band+halo are zero, so any out-of-band read changes the result
        img = np.zeros((rows, cols))
        img[in_row0:in_row0 + in_rows_arr.shape[0]] = in_rows_arr
        out = O.nlem_denoise(img, p, rows=(out_row0, out_row0 + out_rows))
        band = out[out_row0:out_row0 + out_rows]
        assert np.isfinite(band).all()
        return band.astype(np.float32)

    res = D.denoise_bands(noisy, 7, 3, rank, world, band_fn)
    if rank == 0:
        np.save(out_path, res)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_rank_bands_match_single_process(tmp_path, oracle, world):
    rng = np.random.default_rng(5)
    noisy = (rng.uniform(0, 255, size=(23, 17))).astype(np.float32)
    out_path = str(tmp_path / "out.npy")
    mp.spawn(_worker, args=(world, _free_port(), noisy, out_path), nprocs=world, join=True)
    got = np.load(out_path)
    p = oracle.make_params(search=7, patch=3, h=40.0, solver="admm", solver_iters=5, mu=1.0,
                           init_mode="nlm", threads=1)
    ref = oracle.nlem_denoise(noisy.astype(np.float64), p).astype(np.float32)
    assert got.shape == ref.shape
    assert (got == ref).all()


def _gpu_worker(rank, world, port, noisy, out_path):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import paper_1501_03879_b200 as nb

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = nb.NlemParams(search=21, patch=7, h=10 * 20.0 * 7, sigma=20.0, solver="admm",
                      solver_iters=10, mu=1.0, init_mode="nlm")
    # every rank on device 0 (one GPU here); each band goes through the host-buffer C-ABI
    res = D.denoise_bands(noisy, 21, 7, rank, world, D.gpu_band_fn(p, device=0))
    if rank == 0:
        np.save(out_path, res)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_gpu_bands_over_ranks_match_single_call(tmp_path, world):
    """The multi-GPU row-band path with the GPU band function (dist.gpu_band_fn ->
    nlem_denoise_rows_host): world ranks (gloo, all on cuda:0 here), each with its own band
    and 13-row halo, gathered on rank 0 - bitwise equal to one whole-image call."""
    import paper_1501_03879_b200 as nb
    from paper_1501_03879_b200 import synth

    _, noisy = synth.noisy_image(77, 64, 10, 6, 20.0)
    out_path = str(tmp_path / "out.npy")
    mp.spawn(_gpu_worker, args=(world, _free_port(), noisy, out_path), nprocs=world, join=True)
    got = np.load(out_path)
    p = nb.NlemParams(search=21, patch=7, h=10 * 20.0 * 7, sigma=20.0, solver="admm",
                      solver_iters=10, mu=1.0, init_mode="nlm")
    ref = nb.nlem_denoise_host(noisy, p)
    assert got.shape == ref.shape and np.array_equal(got, ref)
