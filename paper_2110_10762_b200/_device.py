"""Device plumbing: torch is the container for device memory and streams
(never the compute path)."""
from __future__ import annotations

import numpy as np
import torch

from . import errors


def require_cuda() -> None:
    if not torch.cuda.is_available():
        raise errors.NativeLibraryError(
            "a CUDA device is required: paper_2110_10762_b200 has no CPU fallback")


def device_index(device=None) -> int:
    require_cuda()
    if device is None:
        return torch.cuda.current_device()
    if isinstance(device, int):
        return device
    d = torch.device(device)
    return d.index if d.index is not None else torch.cuda.current_device()


def stream_ptr(device: int) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def torch_dtype(np_or_str) -> torch.dtype:
    if np_or_str in (np.float32, "float32", "f32", torch.float32):
        return torch.float32
    return torch.float64


def as_device_tensor(x, device: int, dtype: torch.dtype) -> tuple[torch.Tensor, bool]:
    """(tensor on device, was_host). Host inputs are copied H2D; device
    tensors of the right dtype are used as-is (contiguous)."""
    if isinstance(x, torch.Tensor):
        was_host = not x.is_cuda
        t = x.to(device=f"cuda:{device}", dtype=dtype)
        return t.contiguous(), was_host
    arr = np.asarray(x, dtype=np.float64 if dtype == torch.float64 else np.float32)
    t = torch.from_numpy(np.ascontiguousarray(arr)).to(device=f"cuda:{device}", dtype=dtype)
    return t, True


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().to("cpu").numpy()
