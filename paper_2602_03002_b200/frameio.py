"""MDPT depth-frame files and PGM previews.

Same wire formats and API as the reference's frameio.py
(/root/reference/pkg/src/multidepth/frameio.py:1-140):

* MDPT: magic ``MDPT``, u16 version 1, u32 N, C, H, W (little-endian, 22
  header bytes), then N*C*H*W float32 little-endian meters in
  [env][cam][row][col] order (frameio.py:1-8, 21-38). Writing then reading
  reproduces the array bit-exactly.
* PGM P5 previews with depth mapped linearly from [0, d_max] to gray
  [255, 0] (frameio.py:85-91).

B200 side: ``write_frames`` takes the renderer's CUDA observation directly
(one pinned device-to-host copy, then a single write of header + payload);
``depth_to_u8`` runs on the GPU (``mdrt_depth_to_u8``, f64 arithmetic and
round-half-even as numpy, so gray levels are identical); ``FrameWriter``
streams a sequence of frames to disk from a copy stream and a writer thread so
file IO overlaps the following render steps.
"""

from __future__ import annotations

import ctypes
import os
import queue
import struct
import threading

import numpy as np
import torch

from . import _native

MAGIC = b"MDPT"
VERSION = 1
_HEADER = struct.Struct("<4sHIIII")
HEADER_SIZE = _HEADER.size  # 22 bytes


class FormatError(ValueError):
    """Raised when a file does not decode as the expected format (frameio.py:26-27)."""


def _host_f32(data) -> np.ndarray:
    """(N, C, H, W) float32 C-contiguous host array from numpy / torch (CPU or CUDA) / DepthFrame."""
    if hasattr(data, "data") and not isinstance(data, (np.ndarray, torch.Tensor)):
        data = data.data                     # DepthFrame
    if isinstance(data, torch.Tensor):
        t = data.detach()
        if t.device.type == "cuda":
            host = torch.empty(t.shape, dtype=torch.float32, pin_memory=True)
            host.copy_(t.to(torch.float32))
            return host.numpy()
        return np.ascontiguousarray(t.to(torch.float32).numpy())
    return np.ascontiguousarray(data, dtype=np.float32)


def _write_mdpt(path, arr: np.ndarray) -> None:
    if arr.ndim != 4:
        raise ValueError(f"expected (N, C, H, W) data, got shape {arr.shape}")
    n, c, h, w = arr.shape
    with open(path, "wb") as fh:
        fh.write(_HEADER.pack(MAGIC, VERSION, n, c, h, w))
        fh.write(memoryview(arr.astype("<f4", copy=False)).cast("B"))


def write_frames(path, data) -> None:
    """Write an (N, C, H, W) float32 depth batch (frameio.py:30-38)."""
    _write_mdpt(path, _host_f32(data))


def read_frames(path, device=None):
    """Read an MDPT file back to an (N, C, H, W) float32 array (frameio.py:41-62).

    ``device``: None returns numpy (as the reference); a CUDA device returns a
    tensor on it.
    """
    with open(path, "rb") as fh:
        header = fh.read(HEADER_SIZE)
        if len(header) != HEADER_SIZE:
            raise FormatError(f"{path}: truncated header")
        magic, version, n, c, h, w = _HEADER.unpack(header)
        if magic != MAGIC:
            raise FormatError(f"{path}: bad magic {magic!r}")
        if version != VERSION:
            raise FormatError(f"{path}: unsupported version {version}")
        count = n * c * h * w
        payload = fh.read(4 * count)
        if len(payload) != 4 * count:
            raise FormatError(f"{path}: payload holds {len(payload)} bytes, expected {4 * count}")
        if fh.read(1):
            raise FormatError(f"{path}: trailing bytes after payload")
    arr = np.frombuffer(payload, dtype="<f4").reshape(n, c, h, w).astype(np.float32, copy=False)
    if device is None:
        return arr
    return torch.from_numpy(arr.copy()).to(device)


def write_grid(path, grid) -> None:
    """Write a 2-D grid as a 1x1xHxW frame file (frameio.py:65-70)."""
    grid = np.asarray(grid.cpu() if isinstance(grid, torch.Tensor) else grid)
    if grid.ndim != 2:
        raise ValueError(f"expected a 2-D grid, got shape {grid.shape}")
    _write_mdpt(path, np.ascontiguousarray(grid.astype(np.float32)[None, None]))


def read_grid(path) -> np.ndarray:
    """Read a grid written by :func:`write_grid` back to 2-D (frameio.py:73-78)."""
    data = read_frames(path)
    if data.shape[:2] != (1, 1):
        raise FormatError(f"{path}: not a single-grid file (shape {data.shape})")
    return data[0, 0]


def depth_to_u8(depth, d_max: float):
    """Map [0, d_max] depth to 8-bit gray, near = bright (frameio.py:81-86), on the GPU.

    CUDA tensor in -> CUDA uint8 tensor out; numpy / CPU tensor in -> same kind
    out (computed on the GPU).
    """
    if d_max <= 0:
        raise ValueError("d_max must be positive")
    kind = None
    if isinstance(depth, torch.Tensor):
        if depth.device.type != "cuda":
            kind = "torch-cpu"
            t = depth.to("cuda", torch.float32)
        else:
            t = depth.to(torch.float32)
    else:
        kind = "numpy"
        t = torch.from_numpy(np.ascontiguousarray(depth, dtype=np.float32)).cuda()
    t = t.contiguous()
    if t.data_ptr() % 16:
        t = t.clone()
    out = torch.empty(t.shape, dtype=torch.uint8, device=t.device)
    _native.check(_native.lib().mdrt_depth_to_u8(
        ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(out.data_ptr()), t.numel(), float(d_max),
        ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)))
    if kind == "numpy":
        return out.cpu().numpy()
    if kind == "torch-cpu":
        return out.cpu()
    return out


def write_pgm(path, image) -> None:
    """Write an 8-bit grayscale image as binary PGM P5 (frameio.py:89-97)."""
    if isinstance(image, torch.Tensor):
        image = image.cpu().numpy()
    img = np.ascontiguousarray(image)
    if img.ndim != 2 or img.dtype != np.uint8:
        raise ValueError("image must be a 2-D uint8 array")
    h, w = img.shape
    with open(path, "wb") as fh:
        fh.write(f"P5\n{w} {h}\n255\n".encode("ascii"))
        fh.write(img.tobytes())


def read_pgm(path) -> np.ndarray:
    """Read a binary PGM (P5) written by :func:`write_pgm` (frameio.py:100-127)."""
    with open(path, "rb") as fh:
        blob = fh.read()
    fields: list[bytes] = []
    pos, end = 0, len(blob)
    while len(fields) < 4 and pos < end:
        if blob[pos:pos + 1].isspace():
            pos += 1
        elif blob[pos:pos + 1] == b"#":                 # comment to end of line
            nl = blob.find(b"\n", pos)
            pos = end if nl < 0 else nl
        else:
            stop = pos
            while stop < end and not blob[stop:stop + 1].isspace():
                stop += 1
            fields.append(blob[pos:stop])
            pos = stop
    if len(fields) != 4 or fields[0] != b"P5":
        raise FormatError(f"{path}: not a binary PGM")
    w, h, maxval = (int(f) for f in fields[1:])
    if maxval != 255:
        raise FormatError(f"{path}: unsupported maxval {maxval}")
    pos += 1                                            # the single whitespace byte after maxval
    data = blob[pos:pos + w * h]
    if len(data) != w * h:
        raise FormatError(f"{path}: truncated pixel data")
    return np.frombuffer(data, dtype=np.uint8).reshape(h, w)


class FrameWriter:
    """Stream observation batches to ``directory/pattern.format(k)`` MDPT files.

    ``submit(obs)`` (a CUDA (N, C, H, W) float32 tensor) enqueues its copy into
    one of ``depth`` pinned host buffers on a dedicated copy stream, ordered
    after the work already queued on the current stream, and returns at once;
    a writer thread waits for the copy and writes the file. At most ``depth``
    frames are in flight (``submit`` blocks while all buffers are busy).
    ``close()`` drains the queue and re-raises the first IO error. The caller
    must not overwrite ``obs`` before the copy ran: call ``submit`` right after
    the step that produced it and alternate output buffers, or use
    ``render_pipeline(host_out=...)`` and write the host tensor instead.
    """

    def __init__(self, directory, pattern: str = "frame_{:04d}.mdpt", depth: int = 2):
        if depth < 1:
            raise ValueError("depth must be >= 1")
        self.directory = os.fspath(directory)
        os.makedirs(self.directory, exist_ok=True)
        self.pattern = pattern
        self.count = 0
        self._bufs: list[torch.Tensor | None] = [None] * depth
        self._free: queue.Queue = queue.Queue()
        for k in range(depth):
            self._free.put(k)
        self._jobs: queue.Queue = queue.Queue()
        self._error: BaseException | None = None
        self._stream = None
        self._thread = threading.Thread(target=self._run, daemon=True)
        self._thread.start()

    def submit(self, obs) -> str:
        if self._error is not None:
            raise self._error
        path = os.path.join(self.directory, self.pattern.format(self.count))
        self.count += 1
        if not (isinstance(obs, torch.Tensor) and obs.device.type == "cuda"):
            self._jobs.put((None, None, _host_f32(obs), path))
            return path
        if obs.dtype != torch.float32 or obs.dim() != 4:
            raise ValueError("obs must be an (N, C, H, W) float32 CUDA tensor")
        if self._stream is None:
            self._stream = torch.cuda.Stream(obs.device)
        k = self._free.get()
        buf = self._bufs[k]
        if buf is None or tuple(buf.shape) != tuple(obs.shape):
            buf = self._bufs[k] = torch.empty(obs.shape, dtype=torch.float32, pin_memory=True)
        self._stream.wait_stream(torch.cuda.current_stream(obs.device))
        with torch.cuda.stream(self._stream):
            buf.copy_(obs, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self._stream)
        obs.record_stream(self._stream)
        self._jobs.put((k, ev, buf, path))
        return path

    def _run(self):
        while True:
            job = self._jobs.get()
            if job is None:
                return
            k, ev, buf, path = job
            try:
                if ev is not None:
                    ev.synchronize()
                if self._error is None:
                    _write_mdpt(path, buf.numpy() if isinstance(buf, torch.Tensor) else buf)
            except BaseException as exc:  # surfaced by submit/close
                self._error = exc
            finally:
                if k is not None:
                    self._free.put(k)

    def close(self) -> None:
        if self._thread.is_alive():
            self._jobs.put(None)
            self._thread.join()
        if self._error is not None:
            raise self._error

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
