"""MDPT frame files, grids and PGM previews (reference frameio.py), pinned to
bytes written by the live reference (tests/golden/frameio.npz)."""

import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from paper_2602_03002_b200 import frameio


@pytest.fixture(scope="module")
def fio():
    return dict(np.load(os.path.join(GOLDEN, "frameio.npz")))


def test_oracle_matches_reference_vectors(fio):
    from oracle import oracle as orc
    assert orc.mdpt_bytes(fio["depth"]) == fio["mdpt_bytes"].tobytes()
    for k, dmax in enumerate(fio["u8_dmax"]):
        assert np.array_equal(orc.depth_to_u8(fio["depth"], dmax), fio[f"u8_{k}"])


def test_mdpt_bytes_and_round_trip(tmp_path, fio):
    p = tmp_path / "a.mdpt"
    frameio.write_frames(p, fio["depth"])
    assert p.read_bytes() == fio["mdpt_bytes"].tobytes()
    back = frameio.read_frames(p)
    assert back.dtype == np.float32 and np.array_equal(back, fio["depth"])
    frameio.write_frames(p, torch.from_numpy(fio["depth"]))          # CPU tensor
    assert p.read_bytes() == fio["mdpt_bytes"].tobytes()
    g = tmp_path / "g.mdpt"
    frameio.write_grid(g, fio["depth"][1, 1].astype(np.float64))
    assert g.read_bytes() == fio["grid_bytes"].tobytes()
    assert np.array_equal(frameio.read_grid(g), fio["depth"][1, 1])
    with pytest.raises(frameio.FormatError, match="single-grid"):
        frameio.read_grid(p)
    with pytest.raises(ValueError):
        frameio.write_frames(p, np.zeros((2, 3)))
    with pytest.raises(ValueError):
        frameio.write_grid(g, np.zeros((1, 2, 3)))


def test_mdpt_rejects_corrupt_files(tmp_path, fio):
    good = fio["mdpt_bytes"].tobytes()
    cases = {"short": good[:10], "magic": b"XDPT" + good[4:], "version": good[:4] + b"\x02\x00" + good[6:],
             "payload": good[:-4], "trailing": good + b"\x00"}
    for name, blob in cases.items():
        p = tmp_path / f"{name}.mdpt"
        p.write_bytes(blob)
        with pytest.raises(frameio.FormatError):
            frameio.read_frames(p)


def test_pgm_bytes_and_parser(tmp_path, fio):
    img = fio["u8_0"][0, 1]
    p = tmp_path / "p.pgm"
    frameio.write_pgm(p, img)
    assert p.read_bytes() == fio["pgm_bytes"].tobytes()
    assert np.array_equal(frameio.read_pgm(p), img)
    c = tmp_path / "c.pgm"                                         # comments in the header
    c.write_bytes(b"P5\n# made by hand\n3 2\n# max\n255\n" + bytes(range(6)))
    assert np.array_equal(frameio.read_pgm(c), np.arange(6, dtype=np.uint8).reshape(2, 3))
    for blob in (b"P6\n3 2\n255\n" + bytes(6), b"P5\n3 2\n65535\n" + bytes(12), b"P5\n3 2\n255\n" + bytes(5)):
        c.write_bytes(blob)
        with pytest.raises(frameio.FormatError):
            frameio.read_pgm(c)
    with pytest.raises(ValueError):
        frameio.write_pgm(p, img.astype(np.float32))


@pytest.mark.gpu
def test_depth_to_u8_gpu_matches_reference(pkg, fio):
    d = torch.from_numpy(fio["depth"]).cuda()
    for k, dmax in enumerate(fio["u8_dmax"]):
        got = pkg.depth_to_u8(d, float(dmax))
        assert got.is_cuda and got.dtype == torch.uint8
        assert np.array_equal(got.cpu().numpy(), fio[f"u8_{k}"])
    assert np.array_equal(pkg.depth_to_u8(fio["depth"], 10.0), fio["u8_0"])           # numpy in/out
    odd = d.flatten()[3:3 + 1001]                                                       # misaligned, ragged
    assert np.array_equal(pkg.depth_to_u8(odd, 10.0).cpu().numpy(), fio["u8_0"].ravel()[3:3 + 1001])
    with pytest.raises(ValueError):
        pkg.depth_to_u8(d, 0.0)


@pytest.mark.gpu
def test_cuda_frames_and_async_writer(pkg, fio, tmp_path):
    d = torch.from_numpy(fio["depth"]).cuda()
    p = tmp_path / "cuda.mdpt"
    pkg.write_frames(p, d)
    assert p.read_bytes() == fio["mdpt_bytes"].tobytes()
    assert torch.equal(pkg.read_frames(p, device="cuda"), d)
    frames = [d * (k + 1) for k in range(5)]
    with pkg.FrameWriter(tmp_path / "seq", depth=2) as w:
        paths = [w.submit(f) for f in frames]
    for path, f in zip(paths, frames):
        assert np.array_equal(pkg.read_frames(path), f.cpu().numpy())


def test_frame_writer_host_arrays_and_errors(tmp_path, fio):
    """FrameWriter with host arrays (no GPU): files in order, errors surface on close."""
    frames = [fio["depth"] * (k + 1) for k in range(4)]
    with frameio.FrameWriter(tmp_path / "seq", pattern="f_{:02d}.mdpt", depth=2) as w:
        paths = [w.submit(f) for f in frames]
    assert [os.path.basename(p) for p in paths] == [f"f_{k:02d}.mdpt" for k in range(4)]
    for p, f in zip(paths, frames):
        assert np.array_equal(frameio.read_frames(p), f.astype(np.float32))
    w2 = frameio.FrameWriter(tmp_path / "bad")
    w2.submit(np.zeros((2, 3)))          # not (N, C, H, W): the writer thread fails
    with pytest.raises(ValueError):
        w2.close()
    with pytest.raises(ValueError):
        frameio.FrameWriter(tmp_path, depth=0)
