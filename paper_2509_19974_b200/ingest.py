"""Ingestion: the audio formats feeding the path.

Host decode with the reference's semantics and exceptions:
- ``load_wav_bytes``: mono 16-bit PCM WAV to float64 samples pcm / 32768
  (/root/reference/pkg/src/qxcorr/signalgen.py:150-172, via the same
  stdlib ``wave`` parser);
- ``load_raw_bytes``: headerless little-endian float32 that must be finite
  (signalgen.py:189-196).

Device decode for the engine:
- ``wav_to_device``: parse the header on the host, copy only the int16 payload
  (2 B/sample instead of 4) and decode it on the GPU with qx_decode_pcm16 into
  float32. pcm / 32768 is exact in float32, so every quantiser level equals the
  reference's float64 one.
- ``raw_to_device``: validate the bytes on the host (finite float32, as
  load_raw_bytes does) and copy the payload once.
"""

from __future__ import annotations

import ctypes
import io
import wave

import numpy as np

from . import _device as D
from . import _native as N
from ._call import call
from .errors import ParseError, UnsupportedFormat
from .signals import Signal

__all__ = ["load_wav_bytes", "load_raw_bytes", "wav_to_device", "raw_to_device"]


def _wav_frames(data: bytes) -> bytes:
    """The PCM16 payload of a mono WAV, with the reference's checks."""
    try:
        with wave.open(io.BytesIO(data), "rb") as wf:
            channels = wf.getnchannels()
            width = wf.getsampwidth()
            frames = wf.readframes(wf.getnframes())
    except wave.Error as exc:
        if "unknown format" in str(exc):
            raise UnsupportedFormat(f"WAV encoding not supported: {exc}") from exc
        raise ParseError(f"not a readable WAV file: {exc}") from exc
    except EOFError as exc:
        raise ParseError("WAV file is truncated") from exc
    if channels != 1:
        raise UnsupportedFormat(f"expected mono audio, got {channels} channels")
    if width != 2:
        raise UnsupportedFormat(f"expected 16-bit PCM, got {8 * width}-bit")
    if len(frames) < 2:
        raise ParseError("WAV file holds no samples")
    if len(frames) % 2:
        raise ParseError("WAV data chunk is truncated mid-sample")
    return frames


def load_wav_bytes(data: bytes) -> Signal:
    """Mono 16-bit PCM WAV content -> samples in [-1, 1) (signalgen.py:150-172)."""
    return Signal(0, np.frombuffer(_wav_frames(data), dtype="<i2").astype(np.float64) / 32768.0)


def load_raw_bytes(data: bytes) -> Signal:
    """Headerless little-endian float32 stream (signalgen.py:189-196)."""
    if not data or len(data) % 4:
        raise ParseError("raw stream length must be a positive multiple of 4 bytes")
    samples = np.frombuffer(data, dtype="<f4").astype(np.float64)
    if not np.all(np.isfinite(samples)):
        raise ParseError("raw stream contains non-finite values")
    return Signal(0, samples)


def wav_to_device(data: bytes, device=None):
    """float32 CUDA tensor of the WAV's samples: the int16 payload crosses
    PCIe and is decoded by qx_decode_pcm16 (exactly load_wav_bytes' values)."""
    t = D.torch()
    frames = _wav_frames(data)
    pcm = t.frombuffer(bytearray(frames), dtype=t.int16)
    dev = t.device("cuda", device if device is not None else t.cuda.current_device())
    dpcm = pcm.to(dev)
    out = t.empty(pcm.numel(), dtype=t.float32, device=dev)
    call(N.load().qx_decode_pcm16, N.context(dev.index), dpcm.data_ptr(), pcm.numel(), out.data_ptr(),
         D.stream_handle())
    return out


def raw_to_device(data: bytes, device=None):
    """float32 CUDA tensor of a raw little-endian float32 stream.  The
    finiteness check of load_raw_bytes is the format validation of the host
    bytes (numpy, before the upload, as the reference does); the samples then
    cross PCIe once and are not touched again on the host."""
    t = D.torch()
    if not data or len(data) % 4:
        raise ParseError("raw stream length must be a positive multiple of 4 bytes")
    arr = np.frombuffer(data, dtype="<f4")
    if not np.isfinite(arr).all():
        raise ParseError("raw stream contains non-finite values")
    dev = t.device("cuda", device if device is not None else t.cuda.current_device())
    return t.from_numpy(arr.copy()).to(dev)
