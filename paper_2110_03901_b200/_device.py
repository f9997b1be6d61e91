"""Device plumbing for the host-side mirror: array <-> CUDA tensor movement,
dtype routing and 16-byte channel alignment.  PyTorch provides device memory
and streams only; all arithmetic on the path runs in libimconv.so.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

_TORCH_CODE = {torch.bfloat16: _lib.BF16, torch.float16: _lib.F16, torch.int8: _lib.I8,
               torch.float32: _lib.F32, torch.int32: _lib.I32}
_ELEM = {_lib.BF16: 2, _lib.F16: 2, _lib.I8: 1, _lib.F32: 4, _lib.I32: 4}
_CODE_TORCH = {v: k for k, v in _TORCH_CODE.items()}


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the sm_100a convolution has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def is_device_array(a) -> bool:
    return isinstance(a, torch.Tensor) and a.is_cuda


def to_device(a, dtype: torch.dtype | None = None, non_blocking: bool = True) -> torch.Tensor:
    """numpy / CPU tensor / CUDA tensor -> contiguous CUDA tensor (optionally cast)."""
    dev = require_cuda()
    if isinstance(a, torch.Tensor):
        t = a
    else:
        arr = np.ascontiguousarray(np.asarray(a))
        t = torch.from_numpy(arr)
        if non_blocking:
            t = t.pin_memory()
    if not t.is_cuda:
        t = t.to(dev, non_blocking=non_blocking)
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    return t.contiguous()


def to_host(t: torch.Tensor, np_dtype=None) -> np.ndarray:
    out = t.cpu()
    if out.dtype == torch.bfloat16:
        out = out.float()
    arr = out.numpy()
    if np_dtype is not None and arr.dtype != np_dtype:
        arr = arr.astype(np_dtype)
    return arr


def torch_dtype_of(a) -> torch.dtype:
    if isinstance(a, torch.Tensor):
        return a.dtype
    return torch.from_numpy(np.zeros(0, dtype=np.asarray(a).dtype)).dtype


def is_integer_dtype(dt: torch.dtype) -> bool:
    return not (dt.is_floating_point or dt.is_complex or dt == torch.bool)


def aligned_channels(c: int, elem: int) -> int:
    """Smallest channel count >= c whose row is 16, 32, 64 or a multiple of
    128 bytes (the A-tile row widths the TMA/UMMA layouts support)."""
    b = c * elem
    for cand in (16, 32, 64, 128):
        if b <= cand:
            return cand // elem
    return -(-b // 16) * 16 // elem


def aligned_k(k: int, elem: int) -> int:
    step = 16 // elem
    return -(-k // step) * step


def pad_nhwc(x: torch.Tensor, c_pad: int) -> torch.Tensor:
    """(N,H,W,C) -> (N,H,W,C_pad) zero-filled, via imconv_pad_copy."""
    n, h, w, c = x.shape
    if c_pad == c:
        return x
    out = torch.empty((n, h, w, c_pad), dtype=x.dtype, device=x.device)
    _lib.check(_lib.lib.imconv_pad_copy(x.data_ptr(), out.data_ptr(), x.element_size(), n * h * w, 1, c, 1,
                                        c_pad, stream_handle()), "imconv_pad_copy")
    return out


def pad_hwcn(w: torch.Tensor, c_pad: int, k_pad: int) -> torch.Tensor:
    """(R,S,C,K) -> (R,S,C_pad,K_pad) zero-filled, via imconv_pad_copy."""
    r, s, c, k = w.shape
    if c_pad == c and k_pad == k:
        return w
    out = torch.empty((r, s, c_pad, k_pad), dtype=w.dtype, device=w.device)
    _lib.check(_lib.lib.imconv_pad_copy(w.data_ptr(), out.data_ptr(), w.element_size(), r * s, c, k, c_pad,
                                        k_pad, stream_handle()), "imconv_pad_copy")
    return out
