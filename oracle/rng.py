"""Counter-keyed uniforms: SeedSequence -> PCG64 -> double, restated.

The reference draws every random number from
``np.random.default_rng(np.random.SeedSequence(entropy=(seed, seq_id, role,
counter)))`` (ref:sampling.py:53-66) and consumes ``rng.random()`` once per
sample (ref:sampling.py:107-109) — twice for an accept test that rejects
(ref:sampling.py:142-146).  numpy is a third-party dependency (pinned loosely
``numpy>=1.24`` at ref:pyproject.toml:10-13; 2.3.5 here).  Its published
algorithms are restated below in integer Python so the device RNG
(`csrc/rng.cuh`) has an independent, exact specification:

* SeedSequence (O'Neill's seed_seq hash, numpy/random/bit_generator.pyx):
  entropy ints -> little-endian uint32 words -> 4-word pool via ``hashmix`` /
  ``mix`` -> ``generate_state`` words.
* PCG64 (XSL-RR 128/64, numpy/random/src/pcg64): state seeded from the
  first two uint64 of ``generate_state(4, uint64)``, increment from the last
  two; ``next64`` = step, then xor-shift-low + random rotation.
* ``random()`` = ``(next64 >> 11) * 2**-53``.

`tests/test_oracle_rng.py` checks this restatement against numpy itself
and against the golden uniforms produced through the reference's
``RngStream``.
"""

from __future__ import annotations

import numpy as np

M32 = 0xFFFFFFFF
M64 = 0xFFFFFFFFFFFFFFFF
M128 = (1 << 128) - 1

INIT_A = 0x43B0D7E5
MULT_A = 0x931E8875
INIT_B = 0x8B51F9DD
MULT_B = 0x58F38DED
MIX_MULT_L = 0xCA01F9DD
MIX_MULT_R = 0x4973F715
POOL = 4

PCG_MULT = (2549297995355413924 << 64) | 4865540595714422341

ROLE_DRAFT = 0   # ref:sampling.py:20-22
ROLE_VERIFY = 1


def _words(x: int) -> list[int]:
    """One non-negative int -> its little-endian uint32 words ([0] for 0)."""
    if x < 0:
        raise ValueError("entropy must be non-negative")
    if x == 0:
        return [0]
    out = []
    while x:
        out.append(x & M32)
        x >>= 32
    return out


def _hashmix(value: int, hc: list[int]) -> int:
    value ^= hc[0]
    hc[0] = (hc[0] * MULT_A) & M32
    value = (value * hc[0]) & M32
    return value ^ (value >> 16)


def _mix(x: int, y: int) -> int:
    r = (MIX_MULT_L * x - MIX_MULT_R * y) & M32
    return r ^ (r >> 16)


def seedseq_state(entropy: tuple[int, ...], n_words: int) -> list[int]:
    """SeedSequence(entropy).generate_state(n_words, uint32)."""
    ent = []
    for e in entropy:
        ent.extend(_words(int(e)))
    pool = [0] * POOL
    hc = [INIT_A]
    for i in range(POOL):
        pool[i] = _hashmix(ent[i] if i < len(ent) else 0, hc)
    for src in range(POOL):
        for dst in range(POOL):
            if src != dst:
                pool[dst] = _mix(pool[dst], _hashmix(pool[src], hc))
    for src in range(POOL, len(ent)):
        for dst in range(POOL):
            pool[dst] = _mix(pool[dst], _hashmix(ent[src], hc))
    out = []
    hb = INIT_B
    for i in range(n_words):
        v = pool[i % POOL] ^ hb
        hb = (hb * MULT_B) & M32
        v = (v * hb) & M32
        out.append(v ^ (v >> 16))
    return out


def _pcg64_seed(entropy: tuple[int, ...]) -> tuple[int, int]:
    w = seedseq_state(entropy, 8)
    u64 = [w[2 * i] | (w[2 * i + 1] << 32) for i in range(4)]
    initstate = (u64[0] << 64) | u64[1]
    initseq = (u64[2] << 64) | u64[3]
    inc = ((initseq << 1) | 1) & M128
    state = (0 * PCG_MULT + inc) & M128
    state = (state + initstate) & M128
    state = (state * PCG_MULT + inc) & M128
    return state, inc


def _xsl_rr(state: int) -> int:
    x = ((state >> 64) ^ state) & M64
    rot = state >> 122
    return ((x >> rot) | (x << ((64 - rot) & 63))) & M64


def pcg64_uniforms(entropy: tuple[int, ...], n: int) -> list[float]:
    """First ``n`` doubles of default_rng(SeedSequence(entropy)).random()."""
    state, inc = _pcg64_seed(entropy)
    out = []
    for _ in range(n):
        state = (state * PCG_MULT + inc) & M128
        out.append((_xsl_rr(state) >> 11) * (1.0 / 9007199254740992.0))
    return out


def keyed_uniforms(seed: int, seq_id: int, role: int, counter: int,
                   n: int = 2) -> list[float]:
    """Uniforms for one reference key (ref:sampling.py:61-66)."""
    return pcg64_uniforms((int(seed) & M64, int(seq_id), int(role),
                           int(counter)), n)


def numpy_keyed_generator(seed: int, seq_id: int, role: int,
                          counter: int) -> np.random.Generator:
    """The numpy object the reference constructs, for cross-checks."""
    key = (int(seed) & M64, int(seq_id), int(role), int(counter))
    return np.random.default_rng(np.random.SeedSequence(entropy=key))
