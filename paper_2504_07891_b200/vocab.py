"""Synthetic word-level vocabulary obeying the reference's token model.

The reference counts one token per whitespace-delimited unit
(``prompts.py:13-14``) and truncates by re-joining units with spaces
(``prompts.py:17-24``); ``validate_trajectory`` requires a backend's reported
token counts to agree with that count (``engine.py:727-728``).  A device
backend therefore needs a tokenizer whose ids are exactly the whitespace
units of the text.  This module provides one:

* every id renders as one word followed by one whitespace character, so the
  rendering of an id sequence splits back into exactly those ids and
  concatenating renderings never fuses two words;
* ids 0-9 are the digit words ``"0"``..``"9"`` (the judge's score tokens);
  fixed ids hold ``<think>``, ``</think>`` and the verify template's final
  word ``"0-9:"`` (the judge cue, see ``shapes.py``);
* every other id is a six-letter consonant-vowel word; a deterministic
  1-in-``boundary_every`` subset are *boundary* words ending in ``.``, ``!``
  or ``?`` that render with a trailing newline, so they end a reasoning step
  under the default stop markers (``core.py:225``);
* a word outside the vocabulary (template prose, words fused by the engine's
  re-joining, e.g. ``"w3</think>"``) maps by a stable hash into the ordinary
  id range: tokenisation is total and deterministic.

Token classes for device-side stopping are derived per request from the
request's stop strings (``token_classes``).
"""

from __future__ import annotations

import hashlib
from functools import lru_cache

import numpy as np

from .domain import END_THINK_MARKER, THINK_OPEN_MARKER

CONSONANTS = "bcdfghjklmnpqrstvwxz"  # 20
VOWELS = "aeiou"                      # 5
_SYL = [c + v for c in CONSONANTS for v in VOWELS]  # 100 syllables

DIGIT_IDS = tuple(range(10))
THINK_OPEN_ID = 10
END_THINK_ID = 11
JUDGE_CUE_ID = 12
JUDGE_CUE_WORD = "0-9:"
FIRST_WORD_ID = 16

# device token classes (uint8), consumed by the decode stop test
CLASS_PLAIN = 0
CLASS_STOP = 1       # rendering contains a stop string: step ends, token kept
CLASS_END_THINK = 2  # ``</think>``: generation ends, marker dropped
CLASS_MASKED = 3     # never produced (LM-head padding rows)


class Vocab:
    """Word <-> id mapping for ``n_text`` ids (shared by draft and base)."""

    def __init__(self, n_text: int, boundary_every: int = 24) -> None:
        if n_text < FIRST_WORD_ID + 100:
            raise ValueError("vocabulary too small")
        if n_text > FIRST_WORD_ID + 100 ** 3:
            raise ValueError("vocabulary too large for 3-syllable words")
        self.n_text = n_text
        self.boundary_every = boundary_every
        words = [""] * n_text
        seps = [" "] * n_text
        for d in DIGIT_IDS:
            words[d] = str(d)
        words[THINK_OPEN_ID] = THINK_OPEN_MARKER
        words[END_THINK_ID] = END_THINK_MARKER
        words[JUDGE_CUE_ID] = JUDGE_CUE_WORD
        for i in range(13, FIRST_WORD_ID):
            words[i] = f"<r{i}>"
        punct = ".!?"
        for i in range(FIRST_WORD_ID, n_text):
            k = i - FIRST_WORD_ID
            w = _SYL[k // 10000] + _SYL[(k // 100) % 100] + _SYL[k % 100]
            if self.is_boundary_id(i):
                w += punct[(k // boundary_every) % 3]
                seps[i] = "\n"
            words[i] = w
        self.words = words
        self.seps = seps
        self._index = {w: i for i, w in enumerate(words)}
        if len(self._index) != n_text:
            raise AssertionError("vocabulary words are not unique")
        self._render = [w + s for w, s in zip(words, seps)]

    # -- structure -------------------------------------------------------
    def is_boundary_id(self, i: int) -> bool:
        return i >= FIRST_WORD_ID and (i * 2654435761 >> 7) % self.boundary_every == 0

    def ordinary_range(self) -> tuple[int, int]:
        return FIRST_WORD_ID, self.n_text

    # -- text <-> ids ----------------------------------------------------
    def word_id(self, word: str) -> int:
        i = self._index.get(word)
        if i is not None:
            return i
        h = int.from_bytes(hashlib.blake2b(word.encode("utf-8"), digest_size=8).digest(), "little")
        return FIRST_WORD_ID + h % (self.n_text - FIRST_WORD_ID)

    def encode(self, text: str) -> list[int]:
        """One id per whitespace unit (``len(encode(t)) == count_tokens(t)``)."""
        get = self._index.get
        out = []
        for w in text.split():
            i = get(w)
            out.append(i if i is not None else self.word_id(w))
        return out

    def render(self, ids) -> str:
        r = self._render
        return "".join(r[int(i)] for i in ids)

    def render_one(self, i: int) -> str:
        return self._render[int(i)]

    # -- device tables ---------------------------------------------------
    def token_classes(self, stop: tuple[str, ...], n_rows: int) -> np.ndarray:
        """uint8 class per LM-head row for a request's stop strings."""
        return _classes(self, tuple(stop), n_rows)

    def problem(self, n_words: int, seed: int) -> str:
        """Synthetic problem statement: ``n_words`` ordinary, non-boundary words."""
        rng = np.random.default_rng(seed)
        lo, hi = self.ordinary_range()
        out: list[str] = []
        while len(out) < n_words:
            i = int(rng.integers(lo, hi))
            if not self.is_boundary_id(i):
                out.append(self.words[i])
        return " ".join(out)


@lru_cache(maxsize=64)
def _classes(vocab: Vocab, stop: tuple[str, ...], n_rows: int) -> np.ndarray:
    cls = np.full(n_rows, CLASS_MASKED, dtype=np.uint8)
    cls[: vocab.n_text] = CLASS_PLAIN
    if stop:
        for i in range(vocab.n_text):
            r = vocab._render[i]
            if any(m in r for m in stop):
                cls[i] = CLASS_STOP
    cls[END_THINK_ID] = CLASS_END_THINK
    return cls


@lru_cache(maxsize=8)
def shared_vocab(n_text: int) -> Vocab:
    return Vocab(n_text)
