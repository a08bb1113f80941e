"""Ingestion: WAV / raw decode with the reference's
semantics (signalgen.py:150-196; cases after pkg/tests/test_signalgen.py:140-205),
and the device decode feeding the engine."""
import io
import wave

import numpy as np
import pytest

from paper_2509_19974_b200 import ingest as I
from paper_2509_19974_b200.errors import ParseError, UnsupportedFormat


def _wav(frames: bytes, channels=1, width=2, rate=16000) -> bytes:
    buf = io.BytesIO()
    with wave.open(buf, "wb") as wf:
        wf.setnchannels(channels)
        wf.setsampwidth(width)
        wf.setframerate(rate)
        wf.writeframes(frames)
    return buf.getvalue()


def _pcm(n, seed=0):
    rng = np.random.default_rng(seed)
    a = rng.integers(-32768, 32768, size=n).astype("<i2")
    edge = [-32768, 32767, 0, -1][:n]
    a[:len(edge)] = edge
    return a


def test_wav_decode_values():
    pcm = _pcm(1000)
    s = I.load_wav_bytes(_wav(pcm.tobytes()))
    assert s.start == 0 and s.samples.dtype == np.float64
    assert np.array_equal(s.samples, pcm.astype(np.float64) / 32768.0)


def test_wav_errors():
    with pytest.raises(ParseError):
        I.load_wav_bytes(b"RIFF")
    with pytest.raises(ParseError):
        I.load_wav_bytes(b"not audio at all, just text ............")
    with pytest.raises(UnsupportedFormat):
        I.load_wav_bytes(_wav(np.zeros(8, "<i2").tobytes(), channels=2))
    with pytest.raises(UnsupportedFormat):
        I.load_wav_bytes(_wav(np.zeros(8, "<i4").tobytes(), width=4))
    with pytest.raises(ParseError):
        I.load_wav_bytes(_wav(b""))
    # truncated file: header promises more frames than the data chunk holds
    w = bytearray(_wav(np.zeros(64, "<i2").tobytes()))
    with pytest.raises(ParseError):
        I.load_wav_bytes(bytes(w[:40]))


def test_raw_decode_and_errors():
    x = np.random.default_rng(1).standard_normal(33).astype("<f4")
    s = I.load_raw_bytes(x.tobytes())
    assert np.array_equal(s.samples, x.astype(np.float64))
    with pytest.raises(ParseError):
        I.load_raw_bytes(b"")
    with pytest.raises(ParseError):
        I.load_raw_bytes(b"abc")
    with pytest.raises(ParseError):
        I.load_raw_bytes(np.array([1.0, np.nan], "<f4").tobytes())


@pytest.mark.gpu
def test_device_decode_feeds_the_engine():
    """wav_to_device (qx_decode_pcm16) gives exactly load_wav_bytes' values,
    and the engine's estimate on the device-decoded float32 samples equals its
    estimate on the host float64 samples (the reference's representation)."""
    import torch

    import paper_2509_19974_b200 as qx

    for n in (1, 7, 8, 9, 4099, 1 << 16):
        pcm = _pcm(n, seed=n)
        data = _wav(pcm.tobytes())
        d = I.wav_to_device(data)
        assert d.dtype == torch.float32 and d.numel() == n
        assert np.array_equal(d.cpu().numpy().astype(np.float64), I.load_wav_bytes(data).samples)
    sig = np.random.default_rng(3).standard_normal(20000)
    pcm_x = np.clip(np.round(sig[:8192] * 8000), -32768, 32767).astype("<i2")
    pcm_y = np.clip(np.round(sig[300:300 + 4096] * 8000 + 50), -32768, 32767).astype("<i2")
    wx, wy = _wav(pcm_x.tobytes()), _wav(pcm_y.tobytes())
    for q in (qx.sign(), qx.uniform(7, 0.05)):
        dev = qx.estimate_batch(I.wav_to_device(wx), I.wav_to_device(wy), q, q).numpy()[0]
        host = qx.estimate_batch(torch.from_numpy(I.load_wav_bytes(wx).samples.copy()).cuda(),
                                 torch.from_numpy(I.load_wav_bytes(wy).samples.copy()).cuda(), q, q).numpy()[0]
        assert (dev["value"], dev["lag"], dev["ties"]) == (host["value"], host["lag"], host["ties"])
    raw = sig[:1000].astype("<f4").tobytes()
    assert np.array_equal(I.raw_to_device(raw).cpu().numpy(), np.frombuffer(raw, "<f4"))
    with pytest.raises(ParseError):
        I.raw_to_device(np.array([np.inf], "<f4").tobytes())
