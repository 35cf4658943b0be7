"""Output formats of the reference's `gen` command (`cli.py:100-120`), produced
from device buffers.

* ``text``  -- ``"".join(f"{v:.17g}\\n" for v in vals)``: formatted on the GPU
  by `zf_format_g17` (exact 17-digit decimal conversion, byte-identical to
  CPython's '%.17g'), then copied to the host as bytes;
* ``f64le`` -- the raw little-endian float64 values (a device-to-host copy).

`write_values` mirrors `_cmd_gen`: draw ``n`` values in chunks from a sampler
and stream them to a binary sink.
"""

from __future__ import annotations

from . import _lib

FORMATS = ("text", "f64le")
_MAX_TEXT = 24  # bytes per value: '-' + "0.000" + 17 digits + '\n'


def format_g17(x):
    """'%.17g\\n' text of a CUDA float64 tensor, as a CUDA uint8 tensor.

    Raises ValueError if a value lies outside the supported domain
    (0 and 1e-22 <= |v| < 1e17, which holds every sampler output)."""
    import torch
    if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float64):
        raise TypeError("format_g17 needs a CUDA float64 tensor")
    x = x.contiguous().view(-1)
    n = x.numel()
    out = torch.empty(max(1, _MAX_TEXT * n), dtype=torch.uint8, device=x.device)
    words = int(_lib.lib().zf_format_scratch_words(n))
    scratch = torch.zeros(words, dtype=torch.int64, device=x.device)
    with torch.cuda.device(x.device):
        _lib.check(_lib.lib().zf_format_g17(x.data_ptr() if n else None, n, out.data_ptr(),
                                            out.numel(), scratch.data_ptr(),
                                            _lib.stream_handle(x.device)))
    total, bad = (int(v) for v in scratch[:2].cpu())
    if bad:
        raise ValueError(f"{bad} values outside the '%.17g' device formatter's domain")
    return out[:total]


def write_values(sampler, n: int, sink, fmt: str = "text", chunk: int = 1 << 22) -> int:
    """Draw ``n`` values from ``sampler`` and write them to the binary file-like
    ``sink`` in ``fmt``; returns the bytes written."""
    if fmt not in FORMATS:
        raise ValueError(f"unknown format: {fmt!r}")
    if n < 0:
        raise ValueError("n must be >= 0")
    written = 0
    left = n
    while left > 0:
        m = min(chunk, left)
        vals = sampler.fill(m)
        if fmt == "f64le":
            data = vals.cpu().numpy().astype("<f8", copy=False).tobytes()
        else:
            data = format_g17(vals).cpu().numpy().tobytes()
        sink.write(data)
        written += len(data)
        left -= m
    sink.flush()
    return written
