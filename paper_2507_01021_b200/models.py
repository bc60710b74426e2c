"""Model shapes and the pinned token table for the segment-transcription path.

The reference never loads a model: its backend is a modeled sleep or a remote
HTTP client (`pkg/src/dictamux/backend.py:148-277`), and model loading is an
explicit spec non-goal (`SPEC.md:259`). The paper's Listing 1
(`PAPER.md:48-61`) names faster-whisper + CTranslate2; neither is vendored or
installable here, so the shapes below are Whisper's published dimensions and
the token ids follow OpenAI's multilingual tokenizer convention (pinned here,
SURVEY.md §8(c) "Pins to fix in repo config").
"""

from __future__ import annotations

from dataclasses import dataclass, field

SAMPLE_RATE = 16000
N_FFT = 400
HOP = 160
CHUNK_S = 30.0
N_SAMPLES = 480_000            # pad_or_trim window, backend.py:87-99
N_FRAMES = 3000                # mel frames per window
N_CTX = 1500                   # encoder positions
MAX_TARGET_POSITIONS = 448


@dataclass(frozen=True)
class WhisperDims:
    name: str
    d_model: int
    enc_layers: int
    dec_layers: int
    heads: int
    ffn: int
    n_mels: int
    vocab: int
    # token table (OpenAI multilingual convention)
    eot: int = 50257
    sot: int = 50258
    lang_en: int = 50259
    transcribe: int = 50359
    no_timestamps: int = 50363

    @property
    def head_dim(self) -> int:
        return self.d_model // self.heads

    @property
    def prompt(self) -> tuple[int, ...]:
        """Listing 1's `prompt_tokens + [no_timestamps]` (`PAPER.md:57-59`):
        [SOT, en, transcribe, notimestamps]; one prompt per batch
        (`SPEC.md:261`)."""
        return (self.sot, self.lang_en, self.transcribe, self.no_timestamps)

    @property
    def start_of_prev(self) -> int:
        """<|startofprev|> (two ids after <|transcribe|> in the OpenAI layout:
        transcribe, startoflm, startofprev)."""
        return self.transcribe + 2

    def prompt_with_context(self, context: "list[int] | tuple[int, ...]") -> tuple[int, ...]:
        """Whisper's conditioning prompt: <|startofprev|> + previous-text ids +
        the task prompt; the context is cut from the left to fit 224 tokens."""
        context = list(context)[-(224 - 1 - 4):]
        return (self.start_of_prev, *context) + self.prompt if context else self.prompt


WHISPER_TINY = WhisperDims("whisper-tiny", 384, 4, 4, 6, 1536, 80, 51865)
WHISPER_BASE = WhisperDims("whisper-base", 512, 6, 6, 8, 2048, 80, 51865)
WHISPER_LARGE_V3 = WhisperDims("whisper-large-v3", 1280, 32, 32, 20, 5120,
                               128, 51866, transcribe=50360,
                               no_timestamps=50364)

WHISPER_MODELS = {m.name: m for m in (WHISPER_TINY, WHISPER_BASE,
                                      WHISPER_LARGE_V3)}


@dataclass(frozen=True)
class Wav2Vec2Dims:
    """wav2vec2-base CTC shape (BASELINE.json cfg5)."""
    name: str = "wav2vec2-base"
    conv_dim: tuple[int, ...] = (512,) * 7
    conv_kernel: tuple[int, ...] = (10, 3, 3, 3, 3, 2, 2)
    conv_stride: tuple[int, ...] = (5, 2, 2, 2, 2, 2, 2)
    hidden: int = 768
    layers: int = 12
    heads: int = 12
    ffn: int = 3072
    vocab: int = 32
    pos_conv_kernel: int = 128
    pos_conv_groups: int = 16
    blank: int = 0
    ln_eps: float = 1e-5

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads


WAV2VEC2_BASE = Wav2Vec2Dims()


def get_model(name: str):
    if name in WHISPER_MODELS:
        return WHISPER_MODELS[name]
    if name == WAV2VEC2_BASE.name:
        return WAV2VEC2_BASE
    raise KeyError(f"unknown model {name!r}; known: "
                   f"{sorted(WHISPER_MODELS) + [WAV2VEC2_BASE.name]}")


def default_token_cap(duration_s: float) -> int:
    """Per-segment greedy cap used by the cfg2-4 workloads: the sim backend's
    text rate (2.5 words/s, `backend.py:112`) x 1.5 tokens/word, clamped to
    the decoder's context (448 positions minus the 4-token prompt)."""
    import math
    return max(1, min(MAX_TARGET_POSITIONS - 4, math.ceil(3.75 * duration_s)))


def byte_tokens(text: str) -> list[int]:
    """Previous-text ids for a text prompt without tokenizer files (there is no
    network for them): the UTF-8 bytes as the byte-level BPE's single-byte
    tokens -- GPT-2's byte order (bytes_to_unicode: printable ranges first,
    then the remaining bytes), which the Whisper vocabularies keep as ids
    0..255. Unmerged, so longer than the real BPE, but within the vocabulary
    and deterministic."""
    bs = list(range(33, 127)) + list(range(161, 173)) + list(range(174, 256))
    order = bs + [b for b in range(256) if b not in bs]
    rank = {b: i for i, b in enumerate(order)}
    return [rank[b] for b in text.encode("utf-8")]
