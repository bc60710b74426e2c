"""CPU restatement of pad_or_trim + Whisper's log-mel front end (test only).

Order follows Listing 1 (`PAPER.md:50-53`) with the reference's sample-domain
`pad_or_trim` (`pkg/src/dictamux/backend.py:87-99`): int16 -> /32768 ->
zero-pad/trim to 480,000 samples -> STFT -> |X|^2 -> slaney mel -> log10 ->
per-segment clamp -> normalise. Arithmetic restated from transformers 5.5.0:
  * mel bank: `audio_utils.py:263-296` (hertz_to_mel, slaney),
    `:299-332` (mel_to_hertz), `:356-375` (triangular bank), `:453-545`
    (mel_filter_bank; norm="slaney") with the Whisper arguments of
    `feature_extraction_whisper.py:95-103`;
  * STFT + log: `feature_extraction_whisper.py:140-164` (periodic Hann 400,
    hop 160, centre reflect padding, drop the last frame, clamp 1e-10,
    log10, max(x, max-8) per segment, (x+4)/4).
Computed in float64 and returned as float32, so it is a tighter reference
than either the numpy or torch path of the library (documented there as equal
within 1e-5).
"""

from __future__ import annotations

import numpy as np

N_FFT, HOP, N_SAMPLES, N_FRAMES, SR = 400, 160, 480_000, 3000, 16000


def pad_or_trim(samples: np.ndarray, window_s: float = 30.0,
                sample_rate_hz: int = SR) -> np.ndarray:
    """`backend.py:87-99`, restated."""
    target = int(round(window_s * sample_rate_hz))
    if len(samples) == target:
        return samples
    if len(samples) > target:
        return samples[:target]
    out = np.zeros(target, dtype=samples.dtype if len(samples) else np.int16)
    out[:len(samples)] = samples
    return out


def _hz_to_mel(f):
    f = np.asarray(f, np.float64)
    mels = 3.0 * f / 200.0
    logstep = 27.0 / np.log(6.4)
    return np.where(f >= 1000.0, 15.0 + np.log(np.maximum(f, 1e-30) / 1000.0)
                    * logstep, mels)


def _mel_to_hz(m):
    m = np.asarray(m, np.float64)
    f = 200.0 * m / 3.0
    logstep = np.log(6.4) / 27.0
    return np.where(m >= 15.0, 1000.0 * np.exp(logstep * (m - 15.0)), f)


def mel_filters(n_mels: int) -> np.ndarray:
    """[201, n_mels] float64 slaney-normalised triangular bank, 0-8 kHz."""
    n_bins = 1 + N_FFT // 2
    mel_f = np.linspace(_hz_to_mel(0.0), _hz_to_mel(8000.0), n_mels + 2)
    filt_f = _mel_to_hz(mel_f)
    fft_f = np.linspace(0, SR // 2, n_bins)
    diff = np.diff(filt_f)
    slopes = filt_f[None, :] - fft_f[:, None]
    down = -slopes[:, :-2] / diff[:-1]
    up = slopes[:, 2:] / diff[1:]
    fb = np.maximum(0.0, np.minimum(down, up))
    enorm = 2.0 / (filt_f[2:n_mels + 2] - filt_f[:n_mels])
    return fb * enorm[None, :]


def hann_periodic() -> np.ndarray:
    k = np.arange(N_FFT, dtype=np.float64)
    return 0.5 - 0.5 * np.cos(2.0 * np.pi * k / N_FFT)


def log_mel(samples: np.ndarray, n_mels: int = 80) -> np.ndarray:
    """One segment (int16, any length) -> [n_mels, 3000] float32."""
    x = pad_or_trim(np.asarray(samples, dtype=np.int16)).astype(np.float64)
    x = x / 32768.0
    xp = np.pad(x, N_FFT // 2, mode="reflect")
    idx = np.arange(N_FRAMES)[:, None] * HOP + np.arange(N_FFT)[None, :]
    frames = xp[idx] * hann_periodic()[None, :]
    spec = np.abs(np.fft.rfft(frames, axis=1)) ** 2          # [3000, 201]
    mel = spec @ mel_filters(n_mels)                            # [3000, n_mels]
    log_spec = np.log10(np.maximum(mel, 1e-10))
    log_spec = np.maximum(log_spec, log_spec.max() - 8.0)
    return ((log_spec + 4.0) / 4.0).T.astype(np.float32)


def log_mel_batch(segments, n_mels: int = 80) -> np.ndarray:
    return np.stack([log_mel(s, n_mels) for s in segments])
