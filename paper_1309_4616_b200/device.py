"""Device-memory plumbing: PyTorch owns the HBM buffers and streams; the
kernels behind the C ABI only see raw pointers."""

from __future__ import annotations

import numpy as np
import torch


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("expstencil_b200 needs a CUDA device (B200); none is available")
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def is_host(x) -> bool:
    return not isinstance(x, torch.Tensor)


def to_device(x, dtype=torch.float64) -> torch.Tensor:
    """Contiguous CUDA tensor view/copy of x (numpy array or tensor)."""
    if isinstance(x, torch.Tensor):
        if x.device.type != "cuda":
            x = x.to(device())
        if x.dtype != dtype:
            x = x.to(dtype)
        return x.contiguous()
    arr = np.ascontiguousarray(x, dtype=np.float64 if dtype == torch.float64 else None)
    return torch.from_numpy(arr).to(device())


def to_device_z(x) -> torch.Tensor:
    """Contiguous complex128 CUDA tensor of x (real input gets a zero
    imaginary part, like numpy's astype(complex128))."""
    if isinstance(x, torch.Tensor):
        if x.device.type != "cuda":
            x = x.to(device())
        return x.to(torch.complex128).contiguous()
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.complex128)).to(device())


def is_complex_data(x) -> bool:
    return x.is_complex() if isinstance(x, torch.Tensor) else np.iscomplexobj(x)


def like_input(t: torch.Tensor, host: bool):
    """Return t as a numpy array when the caller passed host data."""
    return t.cpu().numpy() if host else t


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def empty(n: int, dtype=torch.float64) -> torch.Tensor:
    return torch.empty(n, dtype=dtype, device=device())


class Workspace:
    """Per-device scratch buffer reused across calls (series partials, the
    two w vectors and the second p vector)."""

    def __init__(self):
        self._buf: dict[int, torch.Tensor] = {}

    def get(self, nbytes: int) -> torch.Tensor:
        dev = torch.cuda.current_device()
        buf = self._buf.get(dev)
        if buf is None or buf.numel() < nbytes:
            self._buf.pop(dev, None)
            buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device())
            self._buf[dev] = buf
        return buf
